"""GPU: the config / CLI front-end (tools/main.cpp:99-206, config.cpp) end to end, and the
coupled run's RunRecord (chronos.cpp:271-289).

* byte-identical output directories on re-run (acceptance.cpp:376-433) for `train` (synchronous
  and coupled, FP32 and bf16) and `stragglers` (coupled sweep);
* the CLI's CSVs are the run_training record of the same config;
* the coupled FM/RM record -- consensus after every L updates, held-out / train loss of the
  averaged model per epoch -- against the oracle's coupled_async run to the same event count
  (its event order is a prefix-stable function of the durations, so the run to (k+1)L events is
  the state at record point k)."""
import filecmp
import os

import numpy as np
import pytest

from paper_2110_11199_b200 import LrSchedule, ModelDesc, Precision, Strategy, StrategyConfig, lr_at, run_training
from paper_2110_11199_b200 import chronos as CH
from paper_2110_11199_b200.cli import EXIT_DIVERGENCE, EXIT_OK, main
from paper_2110_11199_b200.engine import write_csv

pytestmark = pytest.mark.gpu

BLSTM = ("[objective]\nkind = blstm\nlayers = 2\nhidden = 32\nbidirectional = true\ninput_dim = 20\nproj = 16\n"
         "classes = 24\nunroll = 6\nsamples = 60\nprecision = {prec}\n")


def _cfg(tmp_path, name, text):
    p = tmp_path / name
    p.write_text(text)
    return str(p)


def _same_dirs(a, b):
    names = sorted(os.listdir(a))
    assert names == sorted(os.listdir(b)) and names
    _, mismatch, errors = filecmp.cmpfiles(a, b, names, shallow=False)
    assert not mismatch and not errors, mismatch


@pytest.mark.parametrize("prec", ["fp32", "bf16"])
@pytest.mark.parametrize("strategy,coupled", [("ADPSGD_RM", "false"), ("ADPSGD_D1D", "false"), ("ADPSGD_FM", "true")])
def test_train_reruns_are_byte_identical(tmp_path, prec, strategy, coupled):
    text = (f"[run]\nkind = train\nseed = 11\n[engine]\nstrategy = {strategy}\nlearners = 4\nbatch = 4\nepochs = 2\n"
            "[lr]\nbase_lr = 0.05\npeak_lr = 0.05\n" + BLSTM.format(prec=prec) +
            f"[cluster]\ncoupled = {coupled}\ncompute_time = 1\ncomm_pairwise = 0.1\nstraggler_learner = 1\n"
            "straggler_factor = 2\n")
    cfg = _cfg(tmp_path, "run.ini", text)
    outs = [str(tmp_path / f"out{i}") for i in range(2)]
    for o in outs:
        assert main(["train", "--config", cfg, "--out", o]) == EXIT_OK
    _same_dirs(*outs)
    files = set(os.listdir(outs[0]))
    assert {"config.ini", "run.csv", "consensus.csv", "summary.txt"} <= files
    assert ("timing.txt" in files) == (coupled == "true")
    run = open(os.path.join(outs[0], "run.csv")).read().splitlines()
    assert run[0] == "epoch,heldout_loss,lr" and len(run) == 3
    cons = open(os.path.join(outs[0], "consensus.csv")).read().splitlines()
    # 60 samples -> 54 train (10 % held out); ipe = 54 // (4 learners x 4) = 3; 2 epochs
    assert cons[0] == "k,distance" and len(cons) == 1 + 2 * 3
    assert "status = CONVERGED" in open(os.path.join(outs[0], "summary.txt")).read()
    # the resolved config re-runs to the same outputs
    again = str(tmp_path / "again")
    assert main(["train", "--config", os.path.join(outs[0], "config.ini"), "--out", again]) == EXIT_OK
    _same_dirs(outs[0], again)


def test_cli_csv_is_the_run_training_record(tmp_path):
    text = ("[run]\nseed = 5\n[engine]\nstrategy = ADPSGD_RM\nlearners = 3\nbatch = 4\nepochs = 2\n"
            "[lr]\nbase_lr = 0.1\npeak_lr = 0.2\nwarmup_epochs = 1\n" + BLSTM.format(prec="fp32"))
    out = str(tmp_path / "cli")
    assert main(["train", "--config", _cfg(tmp_path, "r.ini", text), "--out", out]) == EXIT_OK
    m = ModelDesc(2, 32, True, 20, 16, 24, 6)
    cfg = StrategyConfig(strategy=Strategy.ADPSGD_RM, learners=3, batch=4, epochs=2, seed=5,
                         lr=LrSchedule(base_lr=0.1, peak_lr=0.2, warmup_epochs=1))
    rec = run_training(cfg, m, None, None, 54, precision=Precision.FP32, synth=(60, 5))
    write_csv(rec, str(tmp_path / "api"))
    for f in ("run.csv", "consensus.csv"):
        assert open(os.path.join(out, f)).read() == open(str(tmp_path / "api" / f)).read()


def test_divergence_exit_code(tmp_path):
    text = ("[run]\nseed = 1\n[engine]\nstrategy = ADPSGD_FM\nlearners = 3\nbatch = 4\nepochs = 3\n"
            "[lr]\nbase_lr = 1e6\npeak_lr = 1e6\n" + BLSTM.format(prec="fp32"))
    out = str(tmp_path / "div")
    assert main(["train", "--config", _cfg(tmp_path, "d.ini", text), "--out", out]) == EXIT_DIVERGENCE
    s = open(os.path.join(out, "summary.txt")).read()
    assert "status = DIVERGED" in s and "divergence_epoch = " in s


def test_stragglers_sweep_reruns_are_byte_identical(tmp_path):
    text = ("[run]\nkind = stragglers\nseed = 11\n[engine]\nstrategy = ADPSGD_FM\nlearners = 4\nbatch = 4\n"
            "epochs = 1\n[lr]\nbase_lr = 0.02\npeak_lr = 0.02\n" + BLSTM.format(prec="bf16") +
            "[cluster]\ncoupled = true\ncomm_pairwise = 0.05\n[stragglers]\nfactors = 5, 100\n"
            "strategies = ADPSGD_FM, ADPSGD_D1D\n")
    cfg = _cfg(tmp_path, "s.ini", text)
    outs = [str(tmp_path / f"s{i}") for i in range(2)]
    for o in outs:
        assert main(["stragglers", "--config", cfg, "--out", o]) == EXIT_OK
    _same_dirs(*outs)
    files = set(os.listdir(outs[0]))
    for name in ("ADPSGD_FM", "ADPSGD_D1D"):
        for stem in ("_baseline_", "_f5_", "_f100_"):
            assert {name + stem + "run.csv", name + stem + "consensus.csv"} <= files
    rows = open(os.path.join(outs[0], "slowdown.csv")).read().splitlines()
    assert rows[0] == "strategy,factor,baseline_s,straggler_s,ratio" and len(rows) == 5
    base = CH.ClusterProfile(learners=4, comm_pairwise=0.05)
    want = CH.slowdown_experiment(Strategy.ADPSGD_D1D, base, [5.0, 100.0], 20)
    assert rows[3].split(",")[4] == "%.17g" % want[0]["ratio"]


M = ModelDesc(layers=1, hidden=16, bidirectional=True, input_dim=10, proj=8, classes=12, unroll=5)


@pytest.mark.parametrize("strategy", [Strategy.ADPSGD_FM, Strategy.ADPSGD_RM])
def test_coupled_record_matches_oracle(oracle_mod, strategy):
    O = oracle_mod
    rng = np.random.default_rng(4)
    feats = rng.normal(size=(40, M.unroll, M.input_dim)).astype(np.float32)
    labels = rng.integers(0, M.classes, size=(40, M.unroll)).astype(np.int32)
    L, train = 4, 36
    cfg = StrategyConfig(strategy=strategy, learners=L, batch=3, epochs=2, seed=31,
                         lr=LrSchedule(base_lr=0.3, peak_lr=0.3, anneal_factor=0.5, anneal_start_epoch=1))
    prof = CH.ClusterProfile(learners=L, compute_time=1.0, comm_pairwise=0.05, stragglers=[(2, 2.5)])
    res = CH.coupled_training(prof, cfg, M, feats, labels, train, precision=Precision.FP32)
    rec = res.record
    ipe = 3
    assert rec.iteration_count == 2 * ipe and len(rec.epochs) == 2 and not rec.diverged
    dur = [max(prof.effective_compute(l), prof.comm_pairwise) for l in range(L)]
    target = 2 * ipe * L
    lrs = [lr_at(cfg.lr, e) for e in range((target - 1) // ipe + 1)]
    od = O.desc(M.layers, M.hidden, 1, M.input_dim, M.proj, M.classes, M.unroll)
    held, tr = np.arange(train, 40, dtype=np.int32), np.arange(train, dtype=np.int32)
    for k in range(2 * ipe):
        ref = O.OracleEngine(od, L, 3, 31, feats, labels, train)
        ref.coupled_async(int(strategy), dur, (k + 1) * L, ipe, lrs)
        W = np.stack([ref.model(l) for l in range(L)], 1)
        cons = np.linalg.norm(W - W.mean(1, keepdims=True), 2)
        assert rec.iterations[k][0] == k and rec.iterations[k][2] == lr_at(cfg.lr, k // ipe)
        assert abs(rec.iterations[k][1] - cons) <= 1e-4 * max(cons, 1e-3), (k, rec.iterations[k][1], cons)
        if (k + 1) % ipe == 0:
            e = (k + 1) // ipe - 1
            avg = W.mean(1)
            h = O.lstm_loss_grad(od, avg, feats, labels, held, want_grad=False)
            t = O.lstm_loss_grad(od, avg, feats, labels, tr, want_grad=False)
            assert rec.epochs[e][0] == e
            assert abs(rec.epochs[e][1] - h) <= 1e-5 * h and abs(rec.epochs[e][2] - t) <= 1e-5 * t
    assert res.total_time > 0
