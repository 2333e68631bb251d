"""GPU: every NCCL call site of the multi-rank data path, executed on one B200 through a world-1
NCCL communicator with ADPSGD_COMM_FORCE=1 (the multi-rank branches are taken although every
learner is local): SDPSGD gradient allreduce (engine.cpp:136-154), D1D weight allreduce launched
on the comm stream before the gradient compute and joined by the update (engine.cpp:173-184,
PAPER.md:220-248), the device barrier before FM / RM peer reads, and the NCCL send / recv gossip
baseline (as self exchanges). Each must leave the learners bit-identical to the communicator-free
single-process path; D1D's allreduce must finish inside the compute window (event timestamps)."""
import numpy as np
import pytest

from paper_2110_11199_b200 import LearnerGroup, ModelDesc, Precision, Strategy, StrategyConfig, nccl_unique_id

pytestmark = pytest.mark.gpu

M = ModelDesc(layers=2, hidden=128, bidirectional=True, input_dim=40, proj=32, classes=64, unroll=21)


def _group(strategy, prec, comm, mode=0):
    rng = np.random.default_rng(3)
    feats = rng.normal(size=(300, M.unroll, M.input_dim)).astype(np.float32)
    labels = rng.integers(0, M.classes, size=(300, M.unroll)).astype(np.int32)
    g = LearnerGroup(M, StrategyConfig(strategy=strategy, learners=3, batch=256, seed=41), precision=prec)
    g.set_dataset(feats, labels, 300)
    if comm:
        g.comm_init(0, 1, nccl_unique_id())
        g.set_gossip_mode(mode)
    return g


CASES = [(Strategy.SDPSGD, 0), (Strategy.ADPSGD_D1D, 0), (Strategy.ADPSGD_FM, 0), (Strategy.ADPSGD_RM, 0),
         (Strategy.ADPSGD_FM, 2), (Strategy.ADPSGD_RM, 2)]


@pytest.mark.parametrize("prec", [Precision.FP32, Precision.BF16])
@pytest.mark.parametrize("strategy,mode", CASES)
def test_forced_nccl_paths_equal_local_path(monkeypatch, strategy, mode, prec):
    monkeypatch.setenv("ADPSGD_COMM_FORCE", "1")
    a = _group(strategy, prec, comm=True, mode=mode)
    monkeypatch.setenv("ADPSGD_COMM_FORCE", "0")
    b = _group(strategy, prec, comm=False)
    for _ in range(3):
        la, lb = a.step(0.2), b.step(0.2)
        assert np.array_equal(la, lb)
        if strategy == Strategy.ADPSGD_D1D:
            st = a.stats()
            # the weight allreduce ran on the comm stream and finished before the gradient
            # compute did (hidden behind it)
            assert 0.0 <= st["comm_start_ms"] <= st["comm_end_ms"] <= st["compute_end_ms"], st
    a.barrier()  # the device barrier (1-float NCCL allreduce) itself
    for j in range(3):
        assert np.array_equal(a.weights(j), b.weights(j)), j
    a.close()
    b.close()
