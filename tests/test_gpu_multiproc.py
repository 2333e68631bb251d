"""GPU: the multi-process FM/RM path (one learner per process, neighbours' weights pulled
through CUDA IPC inside the fused mix kernel) run as 3 processes sharing one B200 with the
CUDA-IPC-only transport (NCCL refuses duplicate devices), against the same 3-learner ring hosted
by one process. The per-learner gradients, pairings and mixing arithmetic are identical, so the
weights must agree bit for bit (FM: engine.cpp:156-171; RM pairing: chronos.cpp:227-235; D1D:
the mean over every learner's w_k read through IPC in learner order, engine.cpp:173-184)."""
import multiprocessing as mp
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

WORLD, STEPS = 3, 3


def _model():
    from paper_2110_11199_b200 import ModelDesc
    return ModelDesc(layers=2, hidden=64, bidirectional=True, input_dim=40, proj=32, classes=48, unroll=7)


def _data(m):
    rng = np.random.default_rng(17)
    return (rng.normal(size=(64, m.unroll, m.input_dim)).astype(np.float32),
            rng.integers(0, m.classes, size=(64, m.unroll)).astype(np.int32))


def _worker(rank, port, strategy, prec, mode, q):
    try:
        os.environ.update({"MASTER_ADDR": "127.0.0.1", "MASTER_PORT": str(port)})
        import torch.distributed as dist
        from paper_2110_11199_b200 import LearnerGroup, Precision, Strategy, StrategyConfig
        dist.init_process_group("gloo", rank=rank, world_size=WORLD)
        m = _model()
        feats, labels = _data(m)
        cfg = StrategyConfig(strategy=Strategy(strategy), learners=WORLD, batch=8, seed=23)
        g = LearnerGroup(m, cfg, precision=Precision(prec), device=0, first_learner=rank, local_learners=1)
        g.set_dataset(feats, labels, 64)
        g.comm_init(rank, WORLD, None)  # CUDA-IPC-only transport
        handles = [None] * WORLD
        dist.all_gather_object(handles, g.export_ipc())
        for r, h in enumerate(handles):
            g.import_ipc(r, r, 1, h)
        g.set_gossip_mode(mode)
        dist.barrier()
        losses = []
        for _ in range(STEPS):
            losses.append(float(g.step(0.1)[0]))
            dist.barrier()  # every rank's w_{k+1} is written before anyone pulls it
        # multi-rank consensus distance (sharded Gram over NVLink-mapped peers + a gloo sum) and
        # the all-learner averaged model (engine.cpp:124-128, 284-289; mixing.cpp:159-180)
        import torch
        from paper_2110_11199_b200.dist import shard_range
        from paper_2110_11199_b200.engine import consensus_from_gram
        b, e = shard_range(g.D, rank, WORLD)
        part = torch.from_numpy(g.consensus_gram(b, e).copy())
        dist.all_reduce(part)
        extra = {"consensus": consensus_from_gram(part.numpy()), "avg": g.averaged_model_all()}
        q.put((rank, losses, g.weights(0), extra))
        dist.barrier()
        g.close()
        dist.destroy_process_group()
    except Exception as e:  # surface worker failures in the parent
        q.put((rank, repr(e), None, None))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


CASES = [(s, p, 0) for s in ("ADPSGD_FM", "ADPSGD_RM", "ADPSGD_D1D") for p in ("FP32", "BF16")] + \
        [("ADPSGD_FM", "FP32", 1), ("ADPSGD_RM", "BF16", 1)]


@pytest.mark.parametrize("strategy_name,prec_name,mode", CASES)
def test_multiprocess_ipc_gossip_equals_single_process_ring(strategy_name, prec_name, mode):
    """mode 0: neighbours read inside the fused mix kernel; mode 1: pulled by the copy engines on
    the comm stream while the gradient is computed, then mixed from local copies."""
    from paper_2110_11199_b200 import LearnerGroup, Precision, Strategy, StrategyConfig
    strategy, prec = int(Strategy[strategy_name]), int(Precision[prec_name])
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, port, strategy, prec, mode, q)) for r in range(WORLD)]
    for p in procs:
        p.start()
    got = {}
    for _ in range(WORLD):
        rank, losses, w, extra = q.get(timeout=300)
        assert w is not None, f"rank {rank} failed: {losses}"
        got[rank] = (losses, w, extra)
    for p in procs:
        p.join(timeout=120)
    m = _model()
    feats, labels = _data(m)
    ref = LearnerGroup(m, StrategyConfig(strategy=Strategy(strategy), learners=WORLD, batch=8, seed=23),
                       precision=Precision(prec))
    ref.set_dataset(feats, labels, 64)
    ref_losses = [ref.step(0.1) for _ in range(STEPS)]
    for r in range(WORLD):
        assert got[r][0] == [float(l[r]) for l in ref_losses], r
        assert np.array_equal(got[r][1], ref.weights(r)), r
    want = ref.consensus_distance()
    avg = ref.averaged_model()
    for r in range(WORLD):
        assert abs(got[r][2]["consensus"] - want) <= 1e-6 * max(want, 1e-12), (r, got[r][2]["consensus"], want)
        assert np.array_equal(got[r][2]["avg"], avg), r
    ref.close()
