#!/usr/bin/env python3
"""Measured slow-learner study (chronos.cpp:142-160 slowdown_experiment, PAPER.md
Table IV): L learner processes (CUDA-IPC transport; round-robin over --gpus devices, default all on GPU 0), learner 0 slowed
by each factor, epoch-time ratio = clean throughput / straggler throughput, measured on real clocks
and set beside the reference's cost-model prediction (chronos.simulate_wallclock).

  FM / RM: free-running asynchronous (adpsgd_async_step, no barrier); throughput = sum of the
           learners' update rates over a fixed wall-clock window.
  D1D:     synchronous mean (adpsgd_step + a host barrier per iteration); throughput = L x K / time.

Every learner has an emulated compute of --compute-ms (host sleep, since the learners may share one
GPU) on top of its real forward/backward; the straggler's (factor - 1) x (real + emulated) compute
is added the same way (adpsgd_set_step_delay / adpsgd_set_straggler).

  python tools/straggler_sweep.py --learners 4 --factors 1 2 5 10 100 > gpurun_out/sweep.json
"""
from __future__ import annotations

import argparse
import json
import multiprocessing as mp
import os
import socket
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def _worker(rank, a, port, q):
    os.environ.update({"MASTER_ADDR": "127.0.0.1", "MASTER_PORT": str(port)})
    import numpy as np
    import torch.distributed as dist
    from paper_2110_11199_b200 import AsyncMode, LearnerGroup, ModelDesc, Precision, Strategy, StrategyConfig
    dist.init_process_group("gloo", rank=rank, world_size=a.learners)
    m = ModelDesc(layers=2, hidden=64, bidirectional=True, input_dim=40, proj=32, classes=64, unroll=21)
    rng = np.random.default_rng(1)
    feats = rng.normal(size=(256, m.unroll, m.input_dim)).astype(np.float32)
    labels = rng.integers(0, m.classes, size=(256, m.unroll)).astype(np.int32)
    dev = rank % a.gpus
    results = []
    for strat in a.strategies:
        for f in a.factors:
            s = Strategy[strat]
            g = LearnerGroup(m, StrategyConfig(strategy=s, learners=a.learners, batch=32, seed=5),
                             precision=Precision.BF16, device=dev, first_learner=rank, local_learners=1)
            g.set_dataset(feats, labels, 256)
            if s != Strategy.ADPSGD_D1D:
                g.async_init(AsyncMode.FREE, 0, 600.0)
            g.comm_init(rank, a.learners, None)
            hs = [None] * a.learners
            dist.all_gather_object(hs, g.export_ipc())
            for r, h in enumerate(hs):
                g.import_ipc(r, r, 1, h)
            g.set_step_delay(0, a.compute_ms, on_host=True)
            if rank == 0:
                g.set_straggler(0, float(f))
            dist.barrier()
            if s == Strategy.ADPSGD_D1D:
                g.step(0.05)
                dist.barrier()
                k = max(3, int(a.window_s * 1000.0 / (a.compute_ms * f)))
                t0 = time.perf_counter()
                for _ in range(k):
                    g.step(0.05)
                    dist.barrier()
                dt, n = time.perf_counter() - t0, k
            else:
                g.async_step(0.05)
                dist.barrier()
                t0, n = time.perf_counter(), 0
                while time.perf_counter() - t0 < a.window_s:
                    g.async_step(0.05)
                    n += 1
                dt = time.perf_counter() - t0
            loss = float(g.eval_loss(g.weights(0), np.arange(64, dtype=np.int32)))
            dist.barrier()
            tot = [None] * a.learners
            dist.all_gather_object(tot, (n, dt, loss))
            g.close()
            if rank == 0:
                results.append({"strategy": strat, "factor": f, "per_learner": tot})
            dist.barrier()
    if rank == 0:
        q.put(results)
    dist.barrier()
    dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--learners", type=int, default=4)
    ap.add_argument("--gpus", type=int, default=1, help="learners are placed round-robin on this many GPUs")
    ap.add_argument("--factors", type=float, nargs="+", default=[1, 2, 5, 10, 100])
    ap.add_argument("--strategies", nargs="+", default=["ADPSGD_FM", "ADPSGD_RM", "ADPSGD_D1D"])
    ap.add_argument("--compute-ms", type=float, default=20.0)
    ap.add_argument("--window-s", type=float, default=3.0)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    from paper_2110_11199_b200 import Strategy
    from paper_2110_11199_b200 import chronos as CH
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    procs = [ctx.Process(target=_worker, args=(r, a, port, q)) for r in range(a.learners)]
    for p in procs:
        p.start()
    res = q.get(timeout=3600)
    for p in procs:
        p.join(timeout=300)
    rows = []
    clean = {}
    for r in res:
        # sum of the learners' own update rates (a learner's last update may overrun the window)
        thr = sum(n / dt for n, dt, _ in r["per_learner"])
        if r["factor"] == 1:
            clean[r["strategy"]] = thr
        rows.append({**r, "throughput_updates_per_s": thr})
    for r in rows:
        s = Strategy[r["strategy"]]
        prof = CH.ClusterProfile(learners=a.learners, compute_time=1.0)
        sim = CH.slowdown_experiment(s, prof, [r["factor"]], 20)[0]["ratio"]
        r["measured_epoch_time_ratio"] = clean[r["strategy"]] / r["throughput_updates_per_s"]
        r["model_epoch_time_ratio"] = sim
        r["straggler_updates"] = r["per_learner"][0][0]
        r["fast_learner_updates_min"] = min(n for n, _, _ in r["per_learner"][1:])
    out = {"tool": "tools/straggler_sweep.py", "learners": a.learners, "gpus": a.gpus, "compute_ms": a.compute_ms,
           "window_s": a.window_s, "transport": "CUDA IPC (one learner per process)",
           "note": "FM/RM free-running async (no barrier); D1D synchronous mean with a host barrier per step; "
                   "emulated compute as host sleeps because the learner processes share the GPU(s)",
           "rows": [{k: v for k, v in r.items() if k != "per_learner"} | {"per_learner": r["per_learner"]} for r in rows]}
    text = json.dumps(out, indent=1)
    print(text)
    if a.out:
        with open(a.out, "w") as f:
            f.write(text + "\n")


if __name__ == "__main__":
    main()
