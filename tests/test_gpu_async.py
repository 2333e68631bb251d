"""GPU: coupled asynchronous FM/RM (chronos.cpp:178-299) on the device vs the oracle's
coupled_async on identical inputs, seeds and durations (event order bit-exact, models within
the FP32 tolerance), and the reference property: homogeneous timing == synchronous engine."""
import numpy as np
import pytest

from paper_2110_11199_b200 import LearnerGroup, ModelDesc, Precision, Strategy, StrategyConfig
from paper_2110_11199_b200 import chronos as CH

pytestmark = pytest.mark.gpu

M = ModelDesc(layers=1, hidden=16, bidirectional=True, input_dim=10, proj=8, classes=12, unroll=5)


def _data(n=40):
    rng = np.random.default_rng(4)
    return (rng.normal(size=(n, M.unroll, M.input_dim)).astype(np.float32),
            rng.integers(0, M.classes, size=(n, M.unroll)).astype(np.int32))


def _odesc(O):
    return O.desc(M.layers, M.hidden, 1, M.input_dim, M.proj, M.classes, M.unroll)


@pytest.mark.parametrize("strategy", [Strategy.ADPSGD_FM, Strategy.ADPSGD_RM])
def test_async_with_straggler_matches_oracle(oracle_mod, strategy):
    O = oracle_mod
    feats, labels = _data()
    L = 5
    g = LearnerGroup(M, StrategyConfig(strategy=strategy, learners=L, batch=3, seed=31), precision=Precision.FP32)
    g.set_dataset(feats, labels, 36)
    ref = O.OracleEngine(_odesc(O), L, 3, 31, feats, labels, 36)
    prof = CH.ClusterProfile(learners=L, compute_time=1.0, comm_pairwise=0.05, stragglers=[(0, 2.5)])
    dur = [max(prof.effective_compute(l), prof.comm_pairwise) for l in range(L)]
    lrs = [0.3, 0.15, 0.1, 0.05, 0.025, 0.0125, 0.01, 0.01]  # a fast learner's rounds run past 2 epochs
    ev, et = CH.async_run(g, strategy, dur, 23, 3, lrs)
    oev, oet = ref.coupled_async(int(strategy), dur, 23, 3, lrs)
    assert ev.tolist() == oev.tolist() and np.array_equal(et, oet)
    assert (ev == 0).sum() < (ev == 1).sum()  # the straggler updates less often
    for l in range(L):
        assert np.max(np.abs(g.weights(l) - ref.model(l))) <= 1e-5


def test_homogeneous_coupled_equals_synchronous(oracle_mod):
    # test_chronos.cpp:131-158: coupled FM/RM with homogeneous timing == run_training
    feats, labels = _data()
    L = 4
    cfg = StrategyConfig(strategy=Strategy.ADPSGD_RM, learners=L, batch=3, seed=2025)
    a = LearnerGroup(M, cfg, precision=Precision.FP32)
    a.set_dataset(feats, labels, 36)
    b = LearnerGroup(M, cfg, precision=Precision.FP32)
    b.set_dataset(feats, labels, 36)
    CH.async_run(a, Strategy.ADPSGD_RM, [1.0] * L, 3 * L, 3, [0.2])
    for _ in range(3):
        b.step(0.2)
    for l in range(L):
        assert np.max(np.abs(a.weights(l) - b.weights(l))) <= 1e-6


def test_async_lr_table_must_cover_every_round():
    # no silent clamp of the epoch index (chronos.cpp:216 uses lr_at(cfg.lr, r / ipe) unbounded)
    from paper_2110_11199_b200.errors import ConfigError
    feats, labels = _data()
    g = LearnerGroup(M, StrategyConfig(strategy=Strategy.ADPSGD_FM, learners=3, batch=3, seed=2), precision=Precision.FP32)
    g.set_dataset(feats, labels, 36)
    with pytest.raises(ConfigError):
        CH.async_run(g, Strategy.ADPSGD_FM, [1.0, 1.0, 5.0], 12, 2, [0.1])


def test_coupled_run_profile_checks():
    feats, labels = _data()
    cfg = StrategyConfig(strategy=Strategy.ADPSGD_FM, learners=4, batch=3, epochs=1, seed=9)
    g = LearnerGroup(M, cfg, precision=Precision.FP32)
    g.set_dataset(feats, labels, 36)
    prof = CH.ClusterProfile(learners=4, compute_time=1.0, comm_pairwise=0.01, stragglers=[(0, 50.0)])
    ev, et, total = CH.coupled_run(prof, cfg, g, 36)
    assert len(ev) == 12 and np.all(np.isfinite(g.averaged_model()))
    with pytest.raises(Exception):
        CH.coupled_run(CH.ClusterProfile(learners=5), cfg, g, 36)
