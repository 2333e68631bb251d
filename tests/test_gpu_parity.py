"""GPU parity of the learner step against the CPU fp64 oracle (same inputs, same seeds),
through the C ABI.

Tolerances (stated):
  * pairing / permutations / sampled batches: bit-exact (index work);
  * FP32 mode (SIMT fp32 GEMMs): loss rel err <= 1e-5, gradient max-abs err <= 2e-5 * max|g|,
    weights after N steps max-abs err <= 1e-5;
  * BF16 mode (tcgen05 bf16 x bf16 -> fp32): gradient relative L2 err <= 5e-2, loss rel err <= 1e-2.
"""
import numpy as np
import pytest
import torch

from paper_2110_11199_b200 import LearnerGroup, MixKind, ModelDesc, Precision, Strategy, StrategyConfig
from paper_2110_11199_b200.errors import StalenessOverflowError, SyncViolationError

pytestmark = pytest.mark.gpu

CASES = {
    "uni2": ModelDesc(layers=2, hidden=16, bidirectional=False, input_dim=12, proj=0, classes=24, unroll=5),
    "bi2p": ModelDesc(layers=2, hidden=16, bidirectional=True, input_dim=20, proj=8, classes=40, unroll=7),
    "bi3p_t21": ModelDesc(layers=3, hidden=32, bidirectional=True, input_dim=36, proj=16, classes=64, unroll=21),
    "odd_in": ModelDesc(layers=2, hidden=24, bidirectional=True, input_dim=13, proj=8, classes=16, unroll=4),
    # edge cases: no recurrence (T = 1: dW_hh = 0), and T = 1 on the fused tcgen05 recurrent path
    "t1": ModelDesc(layers=1, hidden=16, bidirectional=True, input_dim=12, proj=8, classes=10, unroll=1),
    "t1_fused": ModelDesc(layers=2, hidden=64, bidirectional=True, input_dim=40, proj=16, classes=32, unroll=1),
}


def _data(m, n_seg=48, seed=0):
    rng = np.random.default_rng(seed)
    feats = rng.normal(size=(n_seg, m.unroll, m.input_dim)).astype(np.float32)
    labels = rng.integers(0, m.classes, size=(n_seg, m.unroll)).astype(np.int32)
    return feats, labels


def _odesc(O, m):
    return O.desc(m.layers, m.hidden, int(m.bidirectional), m.input_dim, m.proj, m.classes, m.unroll)


@pytest.mark.parametrize("name", list(CASES))
def test_gradient_fp32_matches_oracle(oracle_mod, name):
    O, m = oracle_mod, CASES[name]
    feats, labels = _data(m)
    M = 6
    g = LearnerGroup(m, StrategyConfig(learners=1, batch=M, seed=1), precision=Precision.FP32)
    g.set_dataset(feats, labels, 40)
    rng = np.random.default_rng(7)
    w = rng.normal(0, 0.2, g.D)
    idx = rng.integers(0, 40, size=M).astype(np.int32)
    loss, grad = g.gradient(w, idx)
    oloss, ograd = O.lstm_loss_grad(_odesc(O, m), w, feats, labels, idx)
    assert abs(loss - oloss) <= 1e-5 * abs(oloss)
    assert np.max(np.abs(grad - ograd)) <= 2e-5 * np.max(np.abs(ograd))


@pytest.mark.parametrize("name", ["bi2p", "bi3p_t21"])
def test_gradient_bf16_tensor_core_tolerance(oracle_mod, name):
    O, m = oracle_mod, CASES[name]
    feats, labels = _data(m)
    M = 8
    g = LearnerGroup(m, StrategyConfig(learners=1, batch=M, seed=1), precision=Precision.BF16)
    g.set_dataset(feats, labels, 40)
    rng = np.random.default_rng(9)
    w = rng.normal(0, 0.2, g.D)
    idx = rng.integers(0, 40, size=M).astype(np.int32)
    loss, grad = g.gradient(w, idx)
    oloss, ograd = O.lstm_loss_grad(_odesc(O, m), w, feats, labels, idx)
    rel = np.linalg.norm(grad - ograd) / np.linalg.norm(ograd)
    print(f"bf16 {name}: loss rel err {abs(loss - oloss) / oloss:.2e}, grad rel L2 err {rel:.2e}")
    assert abs(loss - oloss) <= 1e-2 * oloss
    assert rel <= 5e-2


@pytest.mark.parametrize("classes", [24, 264, 296, 512])
def test_fused_softmax_ce_ragged_class_tiles(oracle_mod, classes):
    """The fused output-GEMM + softmax-CE splits each 256-class tile into 32-column chunks over
    two epilogue warps; class counts whose last tile leaves one warp with no valid column
    (C % 256 <= 32) must not poison the log-sum-exp (bf16 tolerance)."""
    O = oracle_mod
    m = ModelDesc(layers=1, hidden=16, bidirectional=True, input_dim=20, proj=16, classes=classes, unroll=6)
    feats, labels = _data(m)
    M = 8
    g = LearnerGroup(m, StrategyConfig(learners=1, batch=M, seed=1), precision=Precision.BF16)
    g.set_dataset(feats, labels, 40)
    rng = np.random.default_rng(5)
    w = rng.normal(0, 0.2, g.D)
    idx = rng.integers(0, 40, size=M).astype(np.int32)
    loss, grad = g.gradient(w, idx)
    g.close()
    oloss, ograd = O.lstm_loss_grad(_odesc(O, m), w, feats, labels, idx)
    assert np.isfinite(loss) and np.all(np.isfinite(grad))
    assert abs(loss - oloss) <= 1e-2 * oloss
    assert np.linalg.norm(grad - ograd) / np.linalg.norm(ograd) <= 5e-2


@pytest.mark.parametrize("force", ["0", "1"])
def test_extra_column_and_streamk_gemms(oracle_mod, monkeypatch, force):
    """ADPSGD_FORCE_EXT=1 routes every eligible weight-gradient GEMM with a bias column through the
    extra row-sum MMA (all-ones N = 16 B operand) and every eligible dgrad GEMM through stream-K
    (CTA pairs splitting tiles along K, partials summed by the tile's k-block-0 owner); the
    gradient must match the oracle (bf16 tolerance) and the default kernels closely."""
    O = oracle_mod
    m = ModelDesc(layers=2, hidden=128, bidirectional=True, input_dim=40, proj=256, classes=520, unroll=5)
    feats, labels = _data(m)
    M = 200  # T * M = 1000 frames: several 256-row pair tiles with a ragged last one
    rng = np.random.default_rng(21)
    idx = rng.integers(0, 40, size=M).astype(np.int32)
    monkeypatch.setenv("ADPSGD_FORCE_EXT", force)
    g = LearnerGroup(m, StrategyConfig(learners=1, batch=M, seed=1), precision=Precision.BF16)
    g.set_dataset(feats, labels, 40)
    w = np.random.default_rng(23).normal(0, 0.1, g.D)
    loss, grad = g.gradient(w, idx)
    g.close()
    oloss, ograd = O.lstm_loss_grad(_odesc(O, m), w, feats, labels, idx)
    assert np.isfinite(loss) and np.all(np.isfinite(grad))
    assert abs(loss - oloss) <= 1e-2 * oloss
    assert np.linalg.norm(grad - ograd) / np.linalg.norm(ograd) <= 5e-2


def test_tail_column_wgrad_and_streamk_extra(oracle_mod, monkeypatch):
    """260 input features (the BASELINE shape's input width): the layer-1 dW_ih GEMM takes one
    256-wide tile per row block and carries features 256..259 plus the bias column on an extra
    N = 16 MMA fed from a K-major copy of those columns, stream-K over every CTA pair. Must match
    the oracle (bf16 tolerance) and the plain ragged-tile kernels (ADPSGD_NO_XTRA=1) to fp32
    summation-order noise."""
    O = oracle_mod
    m = ModelDesc(layers=2, hidden=128, bidirectional=True, input_dim=260, proj=256, classes=520, unroll=11)
    feats, labels = _data(m)
    M = 256  # 2816 frames: the long-K weight gradients split K in two (one-wave split-K)
    idx = np.random.default_rng(41).integers(0, 40, size=M).astype(np.int32)
    w = None
    out = {}
    for noxtra in ("0", "1"):
        monkeypatch.setenv("ADPSGD_NO_XTRA", noxtra)
        g = LearnerGroup(m, StrategyConfig(learners=1, batch=M, seed=1), precision=Precision.BF16)
        g.set_dataset(feats, labels, 40)
        if w is None:
            w = np.random.default_rng(43).normal(0, 0.1, g.D)
        out[noxtra] = g.gradient(w, idx)
        g.close()
    (l0, g0), (l1, g1) = out["0"], out["1"]
    assert np.all(np.isfinite(g0))
    assert abs(l0 - l1) <= 1e-6 * abs(l1)
    assert np.linalg.norm(g0 - g1) / np.linalg.norm(g1) <= 1e-3
    oloss, ograd = O.lstm_loss_grad(_odesc(O, m), w, feats, labels, idx)
    assert abs(l0 - oloss) <= 1e-2 * oloss
    assert np.linalg.norm(g0 - ograd) / np.linalg.norm(ograd) <= 5e-2
    # the layer-1 input-weight block and its bias (first direction) on their own
    H, I = m.hidden, m.input_dim
    wih = slice(0, 4 * H * I)
    b = slice(4 * H * I + 4 * H * H, 4 * H * I + 4 * H * H + 4 * H)
    for sl in (wih, b):
        assert np.linalg.norm(g0[sl] - g1[sl]) / np.linalg.norm(g1[sl]) <= 1e-3


@pytest.mark.parametrize("smax", ["2", "4"])
def test_split_k_weight_gradients_match_unsplit(monkeypatch, smax):
    """Few-tile, long-K weight gradients (dW_proj here: 5 tiles, K = 5376 frames) run one-wave
    split-K: S K-slices per tile on separate CTA pairs, each pair finalising 1/S of the tile's
    columns from the others' fp32 partials (reduce-scatter, slice-order sums). Must equal the
    unsplit kernel (ADPSGD_SPLIT_MAX=1) to fp32 summation-order noise, column block by block."""
    m = ModelDesc(layers=1, hidden=512, bidirectional=True, input_dim=40, proj=256, classes=64, unroll=21)
    rng = np.random.default_rng(1)
    feats = rng.normal(size=(300, m.unroll, m.input_dim)).astype(np.float32)
    labels = rng.integers(0, m.classes, size=(300, m.unroll)).astype(np.int32)
    idx = rng.integers(0, 300, size=256).astype(np.int32)
    out = {}
    w = None
    for s_ in ("1", smax):
        monkeypatch.setenv("ADPSGD_SPLIT_MAX", s_)
        g = LearnerGroup(m, StrategyConfig(learners=1, batch=256, seed=3), precision=Precision.BF16)
        g.set_dataset(feats, labels, 300)
        if w is None:
            w = g.weights(0)
        out[s_] = g.gradient(w, idx)[1]
        g.close()
    H = m.hidden
    off = 2 * (4 * H * m.input_dim + 4 * H * H + 4 * H)
    a = out["1"][off:off + 256 * 2 * H].reshape(256, 2 * H)
    b = out[smax][off:off + 256 * 2 * H].reshape(256, 2 * H)
    for c in range(0, 2 * H, 32):
        blk = (slice(None), slice(c, c + 32))
        assert np.linalg.norm(b[blk] - a[blk]) <= 1e-4 * np.linalg.norm(a[blk]), c
    assert np.linalg.norm(out[smax] - out["1"]) <= 1e-4 * np.linalg.norm(out["1"])


def test_wide_streamk_dgrad_matches_default_kernels(monkeypatch):
    """H = 512: the layer-2 input dgrad (N = 2H = 1024, K = 8H) takes 256 x 512 CTA-pair tiles with
    stream-K under ADPSGD_FORCE_EXT=1; its gradient must agree with the default kernels' (same
    bf16 operands, different fp32 summation order)."""
    m = ModelDesc(layers=2, hidden=512, bidirectional=True, input_dim=40, proj=256, classes=64, unroll=3)
    feats, labels = _data(m)
    M = 96
    idx = np.random.default_rng(31).integers(0, 40, size=M).astype(np.int32)
    out = {}
    for force in ("0", "1"):
        monkeypatch.setenv("ADPSGD_FORCE_EXT", force)
        g = LearnerGroup(m, StrategyConfig(learners=1, batch=M, seed=1), precision=Precision.BF16)
        g.set_dataset(feats, labels, 40)
        w = np.random.default_rng(32).normal(0, 0.05, g.D)
        out[force] = g.gradient(w, idx)
        g.close()
    (l0, g0), (l1, g1) = out["0"], out["1"]
    assert np.all(np.isfinite(g1))
    assert abs(l1 - l0) <= 1e-4 * abs(l0)
    assert np.linalg.norm(g1 - g0) / np.linalg.norm(g0) <= 1e-2


@pytest.mark.parametrize("kq4", ["0", "1"])
def test_persistent_bptt_k_quarters(oracle_mod, monkeypatch, kq4):
    """Persistent BPTT with the K dimension split in halves (256 x 128 tiles, default) or quarters
    (256 x 256 tiles, ADPSGD_BWD_KQ4=1): same gradient as the oracle within bf16 tolerance."""
    O = oracle_mod
    monkeypatch.setenv("ADPSGD_BWD_KQ4", kq4)
    m = ModelDesc(layers=2, hidden=256, bidirectional=True, input_dim=40, proj=16, classes=48, unroll=4)
    feats, labels = _data(m)
    M = 512
    idx = np.random.default_rng(41).integers(0, 40, size=M).astype(np.int32)
    g = LearnerGroup(m, StrategyConfig(learners=1, batch=M, seed=1), precision=Precision.BF16)
    g.set_dataset(feats, labels, 40)
    w = np.random.default_rng(42).normal(0, 0.2, g.D)
    loss, grad = g.gradient(w, idx)
    g.close()
    oloss, ograd = O.lstm_loss_grad(_odesc(O, m), w, feats, labels, idx)
    assert abs(loss - oloss) <= 1e-2 * oloss
    assert np.linalg.norm(grad - ograd) / np.linalg.norm(ograd) <= 5e-2


@pytest.mark.parametrize("bidir,hidden,M,T", [(True, 64, 136, 9), (False, 64, 136, 9), (True, 256, 300, 5),
                                               (False, 128, 260, 4), (True, 128, 256, 6), (True, 256, 512, 4)])
def test_fused_lstm_kernels_match_oracle_and_unfused(oracle_mod, monkeypatch, bidir, hidden, M, T):
    """H % 64 == 0 selects the fused tcgen05 recurrent kernels (cell fwd / bwd in the GEMM
    epilogue); they must agree with the oracle (bf16 tolerance) and with the unfused
    GEMM + pointwise path (same bf16 operands). M > 128 exercises the row mask; H % 128 == 0
    with M > 128 selects the CTA-pair (cta_group::2) kernels, H = 256 gives several unit tiles;
    bidirectional with M % 256 == 0 runs the whole BPTT of a layer in the persistent kernel."""
    O = oracle_mod
    m = ModelDesc(layers=2, hidden=hidden, bidirectional=bidir, input_dim=40, proj=16, classes=48, unroll=T)
    feats, labels = _data(m)
    rng = np.random.default_rng(3)
    idx = rng.integers(0, 40, size=M).astype(np.int32)
    grads = {}
    for fused in ("1", "0"):
        monkeypatch.setenv("ADPSGD_NO_FUSED", "0" if fused == "1" else "1")
        g = LearnerGroup(m, StrategyConfig(learners=1, batch=M, seed=1), precision=Precision.BF16)
        g.set_dataset(feats, labels, 40)
        w = np.random.default_rng(11).normal(0, 0.2, g.D)
        grads[fused] = g.gradient(w, idx)
        g.close()
    oloss, ograd = O.lstm_loss_grad(_odesc(O, m), w, feats, labels, idx)
    (lf, gf), (lu, gu) = grads["1"], grads["0"]
    rel_o = np.linalg.norm(gf - ograd) / np.linalg.norm(ograd)
    rel_u = np.linalg.norm(gf - gu) / np.linalg.norm(gu)
    print(f"fused vs oracle {rel_o:.2e}, fused vs unfused {rel_u:.2e}")
    assert abs(lf - oloss) <= 1e-2 * oloss
    assert rel_o <= 5e-2
    assert rel_u <= 1e-2


def _engine_pair(O, m, strategy, L, M, seed, precision=Precision.FP32, depth=2, cap=1, mix=MixKind.UNIFORM):
    feats, labels = _data(m, seed=seed)
    cfg = StrategyConfig(strategy=strategy, learners=L, batch=M, seed=seed, staleness_cap=cap, generic_mix=mix)
    g = LearnerGroup(m, cfg, precision=precision)
    g.set_dataset(feats, labels, 40)
    ref = O.OracleEngine(_odesc(O, m), L, M, seed, feats, labels, 40, history_depth=depth)
    return g, ref


@pytest.mark.parametrize("strategy", [Strategy.ADPSGD_FM, Strategy.ADPSGD_RM, Strategy.ADPSGD_D1D, Strategy.SDPSGD])
def test_engine_steps_fp32_match_oracle(oracle_mod, strategy):
    O, m = oracle_mod, CASES["bi2p"]
    L, M = 4, 3
    g, ref = _engine_pair(O, m, strategy, L, M, seed=11)
    for k in range(4):
        loss = g.step(0.3)
        assert ref.step(int(strategy), 0.3, k) == 0
        for j in range(L):
            assert abs(loss[j] - ref.last_loss(j)) <= 1e-5 * ref.last_loss(j)
    for j in range(L):
        assert np.max(np.abs(g.weights(j) - ref.model(j))) <= 1e-5


def test_generic_staleness_fp32_matches_oracle(oracle_mod):
    O, m = oracle_mod, CASES["uni2"]
    L, M = 4, 3
    g, ref = _engine_pair(O, m, Strategy.GENERIC, L, M, seed=5, depth=3, cap=2, mix=MixKind.FIXED_RING)
    taus = [0, 1, 2, 1]
    for k in range(4):
        g.step(0.2, taus=taus)
        assert ref.step(int(Strategy.GENERIC), 0.2, k, generic_mix=0, taus=taus) == 0
    for j in range(L):
        assert np.max(np.abs(g.weights(j) - ref.model(j))) <= 1e-5
    with pytest.raises(StalenessOverflowError):
        g.step(0.2, taus=[0, 3, 0, 0])


@pytest.mark.parametrize("strategy", [Strategy.ADPSGD_FM, Strategy.ADPSGD_RM, Strategy.ADPSGD_D1D, Strategy.SDPSGD])
def test_injected_gradient_steps_match_oracle(oracle_mod, strategy):
    O, m = oracle_mod, CASES["uni2"]
    L = 6
    g, ref = _engine_pair(O, m, Strategy.ADPSGD_D1D, L, 2, seed=21)
    # de-synchronise identically first (one real D1D step on both)
    g.step(0.5)
    ref.step(int(Strategy.ADPSGD_D1D), 0.5, 0)
    g2, ref2 = g, ref
    if strategy == Strategy.SDPSGD:  # needs synchronised models
        g2, ref2 = _engine_pair(O, m, Strategy.SDPSGD, L, 2, seed=21)
    else:
        g2.close()
        g2, ref2 = _engine_pair(O, m, strategy, L, 2, seed=21)
        for j in range(L):
            g2.set_weights(j, ref.model(j))
            ref2.set_model(j, ref.model(j))
    rng = np.random.default_rng(4)
    for k in range(3):  # g2 is a fresh context: its iteration counter starts at 0
        G = rng.normal(size=(L, g2.D))
        g2.step_injected(0.1, G)
        assert ref2.step_injected(int(strategy), 0.1, k, G) == 0
    for j in range(L):
        assert np.max(np.abs(g2.weights(j) - ref2.model(j))) <= 2e-6


def test_single_learner_every_strategy_is_sgd(oracle_mod):
    m = CASES["uni2"]
    feats, labels = _data(m)
    ws = []
    for s in Strategy:
        g = LearnerGroup(m, StrategyConfig(strategy=s, learners=1, batch=4, seed=99), precision=Precision.FP32)
        g.set_dataset(feats, labels, 40)
        for _ in range(3):
            g.step(0.05)
        ws.append(g.weights(0))
        g.close()
    for w in ws[1:]:
        assert np.array_equal(w, ws[0])


def test_sdpsgd_sync_violation():
    m = CASES["uni2"]
    feats, labels = _data(m)
    g = LearnerGroup(m, StrategyConfig(strategy=Strategy.SDPSGD, learners=3, batch=2, seed=3), precision=Precision.FP32)
    g.set_dataset(feats, labels, 40)
    w = g.weights(1)
    w[0] += 1e-3
    g.set_weights(1, w)
    with pytest.raises(SyncViolationError):
        g.step(0.1)


def test_host_batch_step_equals_indexed_step(oracle_mod):
    O, m = oracle_mod, CASES["bi2p"]
    feats, labels = _data(m)
    cfg = StrategyConfig(strategy=Strategy.ADPSGD_FM, learners=3, batch=4, seed=8)
    a = LearnerGroup(m, cfg, precision=Precision.FP32)
    a.set_dataset(feats, labels, 40)
    b = LearnerGroup(m, cfg, precision=Precision.FP32)
    b.set_dataset(feats, labels, 40)
    la = a.step(0.2)
    idx = np.stack([O.learner_batches(8, l, 1, 4, 40)[0] for l in range(3)])
    lb = b.step_host_batch(0.2, feats[idx], labels[idx])
    assert np.allclose(la, lb, rtol=0, atol=0)
    for j in range(3):
        assert np.array_equal(a.weights(j), b.weights(j))


def test_prefetched_host_batches_equal_synchronous_copies():
    """Data-loader path: prefetch_host_batch queues the next batch's H2D copy on a copy stream
    (two staging slots) while the current step computes; the steps must equal the plain
    host-batch steps bit for bit, including a prefetch that is skipped (different batch given)."""
    m = ModelDesc(layers=2, hidden=128, bidirectional=True, input_dim=40, proj=64, classes=96, unroll=7)
    rng = np.random.default_rng(9)
    batches = [(rng.normal(size=(64, m.unroll, m.input_dim)).astype(np.float32),
                rng.integers(0, m.classes, size=(64, m.unroll)).astype(np.int32)) for _ in range(5)]
    runs = {}
    for prefetch in (False, True, "plain2"):
        g = LearnerGroup(m, StrategyConfig(learners=1, batch=64, seed=4), precision=Precision.BF16)
        losses = []
        pf = prefetch is True
        if pf:
            g.prefetch_host_batch(*batches[0])
        for i, (f, l) in enumerate(batches):
            if pf and i + 1 < len(batches) and i != 2:
                g.prefetch_host_batch(*batches[i + 1])
            if pf and i == 3:  # batch 3 was not prefetched; a stale prefetch must not be used
                g.prefetch_host_batch(*batches[0])
            losses.append(g.step_host_batch(0.1, f, l)[0])
        runs[prefetch] = (losses, g.weights(0).copy())
        g.close()
    assert runs[False][0] == runs["plain2"][0], ("plain runs differ", runs[False][0], runs["plain2"][0])
    assert runs[False][0] == runs[True][0], ("prefetch differs", runs[False][0], runs[True][0])
    assert np.array_equal(runs[False][1], runs[True][1])


def test_config_s_fixed_ring_fp32(oracle_mod):
    """BASELINE configs[0]: 2-layer LSTM H=256, 40-dim features, 4 learners, FM."""
    O = oracle_mod
    m = ModelDesc(layers=2, hidden=256, bidirectional=False, input_dim=40, proj=0, classes=32, unroll=21)
    g, ref = _engine_pair(O, m, Strategy.ADPSGD_FM, 4, 4, seed=2026)
    for k in range(2):
        g.step(0.5)
        ref.step(int(Strategy.ADPSGD_FM), 0.5, k)
    for j in range(4):
        assert np.max(np.abs(g.weights(j) - ref.model(j))) <= 1e-5


def test_bf16_training_reduces_loss():
    m = ModelDesc(layers=2, hidden=64, bidirectional=True, input_dim=40, proj=32, classes=64, unroll=21)
    g = LearnerGroup(m, StrategyConfig(strategy=Strategy.ADPSGD_RM, learners=3, batch=32, seed=1),
                     precision=Precision.BF16)
    g.synth_dataset(512, 480, seed=3)
    first = g.step(1.0).mean()
    for _ in range(40):
        last = g.step(1.0).mean()
    assert np.isfinite(last) and last < first


def _full_size_grads(layers, weights_round):
    m = ModelDesc(layers=layers, hidden=1024, bidirectional=True, input_dim=260, proj=256, classes=32000, unroll=21)
    M = 256
    rng = np.random.default_rng(101)
    n_seg = 512
    feats = rng.normal(size=(n_seg, m.unroll, m.input_dim)).astype(np.float32)
    labels = rng.integers(0, m.classes, size=(n_seg, m.unroll)).astype(np.int32)
    idx = rng.integers(0, n_seg, size=M).astype(np.int32)
    groups = {}
    for prec in (Precision.BF16, Precision.FP32):
        groups[prec] = LearnerGroup(m, StrategyConfig(learners=1, batch=M, seed=3), precision=prec)
        groups[prec].set_dataset(feats, labels, n_seg)
    w = groups[Precision.FP32].weights(0).copy()  # the engine's own w0 (0.1 N(0,1), engine.cpp:99-116)
    wr = torch.from_numpy(w).to(torch.bfloat16).float().numpy()
    out = {"bf16": groups[Precision.BF16].gradient(wr, idx), "fp32_r": groups[Precision.FP32].gradient(wr, idx)}
    if weights_round:
        out["fp32"] = groups[Precision.FP32].gradient(w, idx)
    for g in groups.values():
        g.close()
    return out


def _rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


@pytest.mark.parametrize("hidden,batch", [(512, 256), (512, 512), (256, 256)])
def test_paper_widths_bf16_gradient_matches_fp32_engine(hidden, batch):
    """BASELINE's paper shape P uses 512 units/direction: the persistent recurrent kernels at
    H = 512 (and 256) with one or two 256-row blocks per direction, against the FP32 engine on the
    same bf16-representable weights (2 layers, T = 21)."""
    m = ModelDesc(layers=2, hidden=hidden, bidirectional=True, input_dim=260, proj=256, classes=2000, unroll=21)
    rng = np.random.default_rng(5)
    n_seg = 600
    feats = rng.normal(size=(n_seg, m.unroll, m.input_dim)).astype(np.float32)
    labels = rng.integers(0, m.classes, size=(n_seg, m.unroll)).astype(np.int32)
    idx = rng.integers(0, n_seg, size=batch).astype(np.int32)
    out, w = {}, None
    for prec in (Precision.FP32, Precision.BF16):
        g = LearnerGroup(m, StrategyConfig(learners=1, batch=batch, seed=3), precision=prec)
        g.set_dataset(feats, labels, n_seg)
        if w is None:
            w = torch.from_numpy(g.weights(0).copy()).to(torch.bfloat16).float().numpy()
        out[prec] = g.gradient(w, idx)
        g.close()
    (lf, gf), (lb, gb) = out[Precision.FP32], out[Precision.BF16]
    assert np.isfinite(lb) and np.all(np.isfinite(gb))
    assert abs(lb - lf) <= 1e-2 * abs(lf)
    assert _rel(gb, gf) <= 5e-2, _rel(gb, gf)


def test_full_width_two_layer_bf16_gradient_matches_fp32_engine():
    """BASELINE configs[1] widths (1024 units/dir, proj 256, 32k classes, T = 21, 256 segments) at
    2 layers: bf16 tcgen05 path (persistent recurrent kernels, fused 32k-class softmax-CE,
    stream-K / extra-column GEMMs) against the FP32 SIMT engine on the same bf16-representable
    weights. Bar: loss rel err <= 1e-2, gradient rel L2 err <= 5e-2 (bf16 operands; measured 1.7e-2)."""
    out = _full_size_grads(2, False)
    (lb, gb), (lf, gf) = out["bf16"], out["fp32_r"]
    assert np.isfinite(lb) and np.all(np.isfinite(gb))
    assert abs(lb - lf) <= 1e-2 * abs(lf)
    assert _rel(gb, gf) <= 5e-2


def test_full_size_bf16_gradient_at_fp32_conditioning_floor():
    """Full BASELINE configs[1] model (6 layers). With the reference's init (0.1 N(0,1) at 1024
    units, recurrent gain ~3) the 6-layer objective is ill-conditioned: rounding the weights to
    bf16 alone moves the FP32 engine's gradient by ~48 % (measured; tools/fullsize_sens.py), so a
    fixed tolerance is meaningless. Property instead: the bf16 path's distance from the FP32
    engine (same rounded weights) is no larger than 1.5x the FP32 engine's own sensitivity to a
    bf16-sized weight perturbation, and the loss agrees to 1e-2."""
    out = _full_size_grads(6, True)
    (lb, gb), (lr, gr), (lf, gf) = out["bf16"], out["fp32_r"], out["fp32"]
    assert np.isfinite(lb) and np.all(np.isfinite(gb))
    assert abs(lb - lr) <= 1e-2 * abs(lr)
    floor = _rel(gr, gf)
    assert _rel(gb, gr) <= 1.5 * floor + 2e-2, (_rel(gb, gr), floor)


def test_single_segment_batch_and_errors(oracle_mod):
    """Edge cases of the reference's input checks: a one-segment batch matches the oracle;
    stepping without a dataset and a zero batch raise InvalidStateError / ConfigError
    (objectives.cpp:240-241, engine.cpp:60-77)."""
    from paper_2110_11199_b200.errors import AdpsgdError, InvalidStateError
    O, m = oracle_mod, CASES["bi2p"]
    feats, labels = _data(m)
    g = LearnerGroup(m, StrategyConfig(learners=1, batch=1, seed=1), precision=Precision.FP32)
    with pytest.raises(InvalidStateError):
        g.step(0.1)
    g.set_dataset(feats, labels, 40)
    w = np.random.default_rng(3).normal(0, 0.2, g.D)
    idx = np.array([17], dtype=np.int32)
    loss, grad = g.gradient(w, idx)
    oloss, ograd = O.lstm_loss_grad(_odesc(O, m), w, feats, labels, idx)
    assert abs(loss - oloss) <= 1e-5 * abs(oloss)
    assert np.max(np.abs(grad - ograd)) <= 2e-5 * np.max(np.abs(ograd))
    g.close()
    with pytest.raises((AdpsgdError, ValueError)):
        StrategyConfig(learners=1, batch=0, seed=1).validate()
