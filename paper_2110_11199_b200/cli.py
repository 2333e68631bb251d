"""Command-line front-end (proj/tools/main.cpp:99-285): `train` and `stragglers` from a config
file, writing the reference's output files; `python -m paper_2110_11199_b200 <command> ...`.

  train       config.ini (resolved), run.csv (epoch,heldout_loss,lr), consensus.csv (k,distance),
              summary.txt, and timing.txt for coupled runs                    (main.cpp:107-152)
  stragglers  config.ini, slowdown.csv (strategy,factor,baseline_s,straggler_s,ratio) from the
              cluster cost model; with cluster.coupled = true also the coupled runs' CSVs
              <STRATEGY>_baseline_* and <STRATEGY>_f<factor>_*                 (main.cpp:154-206)

Floats are written at 17 significant digits. Exit codes: 0 ok, 2 usage / config error,
3 divergence (main.cpp:26-29). The reference's analyze-mixing and verify commands (spectral
theory battery) are outside this build and exit 2.
"""
from __future__ import annotations

import argparse
import math
import os
import sys

EXIT_OK, EXIT_USAGE, EXIT_DIVERGENCE = 0, 2, 3


def _ensure_out_dir(out: str) -> None:
    from .errors import ConfigError
    try:
        os.makedirs(out, exist_ok=True)
    except OSError:
        raise ConfigError("cannot create output directory: " + out) from None


def _load(args):
    from .config import RunConfig
    config = RunConfig.parse_file(args.config)
    if args.seed is not None:
        config.seed = args.seed % (1 << 64)
        config.strategy.seed = config.seed
    return config


def _write(path: str, text: str) -> None:
    with open(path, "w") as f:
        f.write(text)


def _fmt_factor(f: float) -> str:
    """`stem << name << "_f" << factor` (main.cpp:197): default ostream precision (6, %g)."""
    return "%g" % f


def cmd_train(args) -> int:
    from .chronos import coupled_training
    from .engine import fmt_double, run_training, strategy_name, write_csv
    config = _load(args)
    config.strategy.validate()
    config.cluster.validate()
    _ensure_out_dir(args.out)
    _write(os.path.join(args.out, "config.ini"), config.resolved_text())
    ob = config.objective
    model, prec, train_count = ob.model(), ob.precision_enum(), ob.train_count()
    synth = (ob.samples, config.seed)
    if config.coupled:
        res = coupled_training(config.cluster, config.strategy, model, None, None, train_count, precision=prec,
                               device=args.device, synth=synth)
        record = res.record
        _write(os.path.join(args.out, "timing.txt"), f"total_time = {fmt_double(res.total_time)}\n")
    else:
        record = run_training(config.strategy, model, None, None, train_count, precision=prec, device=args.device,
                              synth=synth)
    write_csv(record, args.out)
    final = record.epochs[-1][1] if record.epochs else math.nan
    lines = [f"strategy = {strategy_name(config.strategy.strategy)}", f"iterations = {record.iteration_count}",
             f"final_heldout_loss = {fmt_double(final)}", f"diverged = {'true' if record.diverged else 'false'}"]
    if record.diverged:
        lines.append(f"divergence_epoch = {record.divergence_epoch}")
    lines.append(f"status = {'DIVERGED' if record.diverged else 'CONVERGED'}")
    _write(os.path.join(args.out, "summary.txt"), "\n".join(lines) + "\n")
    return EXIT_DIVERGENCE if record.diverged else EXIT_OK


def cmd_stragglers(args) -> int:
    from dataclasses import replace
    from .chronos import coupled_training, slowdown_experiment
    from .engine import fmt_double, strategy_name, write_csv
    config = _load(args)
    config.cluster.validate()
    _ensure_out_dir(args.out)
    _write(os.path.join(args.out, "config.ini"), config.resolved_text())
    base = replace(config.cluster, stragglers=[])
    rows = ["strategy,factor,baseline_s,straggler_s,ratio"]
    for s in config.straggler_strategies:
        for r in slowdown_experiment(s, base, config.straggler_factors, config.iterations_per_learner):
            rows.append(",".join([strategy_name(s), fmt_double(r["factor"]), fmt_double(r["baseline_epoch_time"]),
                                  fmt_double(r["straggler_epoch_time"]), fmt_double(r["ratio"])]))
    _write(os.path.join(args.out, "slowdown.csv"), "\n".join(rows) + "\n")
    any_diverged = False
    if config.coupled:
        ob = config.objective
        model, prec, train_count = ob.model(), ob.precision_enum(), ob.train_count()
        synth = (ob.samples, config.seed)
        for s in config.straggler_strategies:
            cfg = replace(config.strategy, strategy=s)
            cfg.validate()
            name = strategy_name(s)
            res = coupled_training(base, cfg, model, None, None, train_count, precision=prec, device=args.device,
                                   synth=synth)
            write_csv(res.record, args.out, name + "_baseline_")
            any_diverged |= res.record.diverged
            for f in config.straggler_factors:
                prof = replace(base, stragglers=[(0, f)])
                res = coupled_training(prof, cfg, model, None, None, train_count, precision=prec,
                                       device=args.device, synth=synth)
                write_csv(res.record, args.out, f"{name}_f{_fmt_factor(f)}_")
                any_diverged |= res.record.diverged
    return EXIT_DIVERGENCE if any_diverged else EXIT_OK


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(
        prog="python -m paper_2110_11199_b200",
        description="ADPSGD on B200: training runs and the straggler sweep from a config file.\n"
                    "CSV columns (floats at 17 significant digits):\n"
                    "  run.csv:       epoch,heldout_loss,lr\n"
                    "  consensus.csv: k,distance\n"
                    "  slowdown.csv:  strategy,factor,baseline_s,straggler_s,ratio\n"
                    "Exit codes: 0 ok, 2 usage/config error, 3 divergence.",
        formatter_class=argparse.RawDescriptionHelpFormatter)
    sub = ap.add_subparsers(dest="cmd")
    for name, help_ in (("train", "One training run from a config file"),
                        ("stragglers", "Straggler slowdown sweep from a config file")):
        p = sub.add_parser(name, help=help_)
        p.add_argument("--config", required=True, help="Run configuration file")
        p.add_argument("--seed", type=int, default=None, help="Override the config seed")
        p.add_argument("--out", default=".", help="Output directory")
        p.add_argument("--device", type=int, default=0, help="CUDA device")
    for name in ("analyze-mixing", "verify"):
        sub.add_parser(name, help="not part of this build (spectral theory battery)", add_help=False)
    try:
        args, extra = ap.parse_known_args(argv)
    except SystemExit as e:
        return EXIT_OK if e.code == 0 else EXIT_USAGE
    if args.cmd is None:
        ap.print_usage(sys.stderr)
        return EXIT_USAGE
    if args.cmd in ("analyze-mixing", "verify"):
        print(f"error: '{args.cmd}' (spectral theory battery) is outside this build", file=sys.stderr)
        return EXIT_USAGE
    if extra:
        print("error: unrecognized arguments: " + " ".join(extra), file=sys.stderr)
        return EXIT_USAGE
    from .errors import ConfigError
    try:
        return cmd_train(args) if args.cmd == "train" else cmd_stragglers(args)
    except ConfigError as e:
        print(f"config error: {e}", file=sys.stderr)
        return EXIT_USAGE
    except Exception as e:  # noqa: BLE001 -- main.cpp:278-281
        print(f"error: {e}", file=sys.stderr)
        return EXIT_USAGE


if __name__ == "__main__":
    sys.exit(main())
