"""GPU: the single-process multi-GPU drop-in (adpsgd_group_link / adpsgd_group_step): learners
spread over several contexts of ONE process -- one per GPU in deployment; here all on the one
B200 -- reading each other's models (and SDPSGD gradients) in place, the contexts' gradient
computes running concurrently. Must equal the single-context ring bit for bit for every strategy
(engine.cpp:136-204, run_training's loop engine.cpp:212-304), with the all-learner consensus
distance (sharded Gram, mixing.cpp:159-180) and averaged model (engine.cpp:124-128)."""
import numpy as np
import pytest

from paper_2110_11199_b200 import DeviceGroup, LearnerGroup, ModelDesc, Precision, Strategy, StrategyConfig

pytestmark = pytest.mark.gpu

M = ModelDesc(layers=2, hidden=64, bidirectional=True, input_dim=40, proj=32, classes=48, unroll=7)


def _data():
    rng = np.random.default_rng(8)
    return (rng.normal(size=(64, M.unroll, M.input_dim)).astype(np.float32),
            rng.integers(0, M.classes, size=(64, M.unroll)).astype(np.int32))


@pytest.mark.parametrize("prec", [Precision.FP32, Precision.BF16])
@pytest.mark.parametrize("strategy", [Strategy.ADPSGD_FM, Strategy.ADPSGD_RM, Strategy.ADPSGD_D1D, Strategy.SDPSGD])
@pytest.mark.parametrize("shares", [[1, 1, 1, 1], [2, 1, 1]])
def test_device_group_equals_single_context(strategy, prec, shares):
    feats, labels = _data()
    cfg = StrategyConfig(strategy=strategy, learners=4, batch=8, seed=19)
    grp = DeviceGroup(M, cfg, devices=[0] * len(shares), precision=prec, shares=shares)
    grp.set_dataset(feats, labels, 64)
    ref = LearnerGroup(M, cfg, precision=prec)
    ref.set_dataset(feats, labels, 64)
    for _ in range(3):
        la, lb = grp.step(0.2), ref.step(0.2)
        assert np.array_equal(la, lb)
    for j in range(4):
        assert np.array_equal(grp.weights(j), ref.weights(j)), j
    want = ref.consensus_distance()
    got = grp.consensus_distance()
    assert abs(got - want) <= 1e-6 * max(want, 1e-12), (got, want)
    assert np.array_equal(grp.averaged_model(), ref.averaged_model())
    grp.close()
    ref.close()
