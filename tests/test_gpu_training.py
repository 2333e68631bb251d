"""GPU: the training loop layer (engine.cpp:206-304) — run_training's iteration / epoch record,
device consensus distance (mixing.cpp:159-180) and forward-only loss evaluation — against the
fp64 oracle driven through the same iteration sequence. FP32 mode, tolerances as in
test_gpu_parity.py."""
import numpy as np
import pytest

from paper_2110_11199_b200 import (LearnerGroup, LrSchedule, ModelDesc, Precision, Strategy, StrategyConfig,
                                   iterations_per_epoch, lr_at, run_training, write_csv)

pytestmark = pytest.mark.gpu

M = ModelDesc(layers=2, hidden=16, bidirectional=True, input_dim=10, proj=8, classes=12, unroll=6)


def _data(n=40, seed=0):
    rng = np.random.default_rng(seed)
    return (rng.normal(size=(n, M.unroll, M.input_dim)).astype(np.float32),
            rng.integers(0, M.classes, size=(n, M.unroll)).astype(np.int32))


def _odesc(O):
    return O.desc(M.layers, M.hidden, 1, M.input_dim, M.proj, M.classes, M.unroll)


def _consensus(ws):
    W = np.stack(ws, 1)
    Dv = W - W.mean(1, keepdims=True)
    return np.linalg.norm(Dv, 2)


@pytest.mark.parametrize("strategy", [Strategy.ADPSGD_RM, Strategy.ADPSGD_D1D])
def test_run_training_matches_oracle(oracle_mod, strategy, tmp_path):
    O = oracle_mod
    feats, labels = _data()
    train = 32
    cfg = StrategyConfig(strategy=strategy, learners=4, batch=2, epochs=2, seed=77,
                         lr=LrSchedule(base_lr=0.2, peak_lr=0.4, warmup_epochs=1))
    rec = run_training(cfg, M, feats, labels, train, precision=Precision.FP32)
    ipe = iterations_per_epoch(cfg, train)
    assert ipe == 4 and rec.iteration_count == 8 and len(rec.epochs) == 2 and not rec.diverged
    # oracle: same iteration sequence
    ref = O.OracleEngine(_odesc(O), 4, 2, 77, feats, labels, train)
    k = 0
    for epoch in range(2):
        lr = lr_at(cfg.lr, epoch)
        for _ in range(ipe):
            assert ref.step(int(strategy), lr, k) == 0
            cons = _consensus([ref.model(l) for l in range(4)])
            assert rec.iterations[k][0] == k and rec.iterations[k][2] == lr
            assert abs(rec.iterations[k][1] - cons) <= 1e-4 * max(cons, 1e-3)
            k += 1
        avg = np.mean([ref.model(l) for l in range(4)], 0)
        held = O.lstm_loss_grad(_odesc(O), avg, feats, labels, np.arange(train, 40, dtype=np.int32), want_grad=False)
        tr = O.lstm_loss_grad(_odesc(O), avg, feats, labels, np.arange(train, dtype=np.int32), want_grad=False)
        assert abs(rec.epochs[epoch][1] - held) <= 1e-5 * held
        assert abs(rec.epochs[epoch][2] - tr) <= 1e-5 * tr
    assert np.max(np.abs(rec.final_model - np.mean([ref.model(l) for l in range(4)], 0))) <= 1e-5
    write_csv(rec, str(tmp_path))
    lines = (tmp_path / "run.csv").read_text().splitlines()
    assert lines[0] == "epoch,heldout_loss,lr" and len(lines) == 3
    assert float(lines[1].split(",")[1]) == rec.epochs[0][1]  # %.17g round-trips


def test_divergence_is_recorded_not_thrown():
    feats, labels = _data()
    cfg = StrategyConfig(strategy=Strategy.SDPSGD, learners=2, batch=4, epochs=6, seed=3,
                         lr=LrSchedule(base_lr=400.0, peak_lr=400.0))
    rec = run_training(cfg, M, feats, labels, 32, precision=Precision.FP32, eval_train=False)
    assert rec.diverged and rec.divergence_epoch >= 0
    assert len(rec.epochs) == rec.divergence_epoch + 1


def test_eval_loss_chunks_and_masks(oracle_mod):
    O = oracle_mod
    feats, labels = _data()
    g = LearnerGroup(M, StrategyConfig(learners=1, batch=4, seed=1), precision=Precision.FP32)
    g.set_dataset(feats, labels, 40)
    w = np.random.default_rng(2).normal(0, 0.3, g.D)
    idx = np.array([3, 9, 1, 22, 30, 5, 17], dtype=np.int32)  # 7 = one full chunk + masked tail
    got = g.eval_loss(w, idx)
    want = O.lstm_loss_grad(_odesc(O), w, feats, labels, idx, want_grad=False)
    assert abs(got - want) <= 1e-5 * want


def test_consensus_distance_bf16_group():
    feats, labels = _data()
    cfg = StrategyConfig(strategy=Strategy.ADPSGD_FM, learners=5, batch=4, seed=9)
    g = LearnerGroup(ModelDesc(layers=1, hidden=64, bidirectional=True, input_dim=10, proj=16, classes=16, unroll=6),
                     cfg, precision=Precision.BF16)
    rng = np.random.default_rng(0)
    ws = [rng.normal(0, 0.1, g.D) for _ in range(5)]
    for j, w in enumerate(ws):
        g.set_weights(j, w)
    want = _consensus([w.astype(np.float32).astype(np.float64) for w in ws])
    assert abs(g.consensus_distance() - want) <= 1e-5 * want


@pytest.mark.parametrize("strategy", [Strategy.ADPSGD_RM, Strategy.ADPSGD_D1D])
def test_bf16_steps_bit_identical_across_runs(strategy):
    """Two engines with the same seed and data produce bit-identical weights after several bf16
    steps (the reference's run_training determinism, test_engine.cpp:344-365): every reduction on
    the path -- stream-K and split-K partial sums, the CE log-sum-exp, bias column sums -- runs in
    a fixed order, and the persistent kernels use atomics only for their step counters."""
    m = ModelDesc(layers=2, hidden=128, bidirectional=True, input_dim=40, proj=256, classes=304, unroll=5)
    cfg = StrategyConfig(strategy=strategy, learners=3, batch=256, seed=11)
    out = []
    for _ in range(2):
        g = LearnerGroup(m, cfg, precision=Precision.BF16)
        g.synth_dataset(1024, 1000, seed=5)
        losses = [g.step(0.5).copy() for _ in range(3)]
        out.append((np.stack(losses), [g.weights(j) for j in range(3)]))
        g.close()
    (l0, w0), (l1, w1) = out
    assert np.array_equal(l0, l1)
    for a, b in zip(w0, w1):
        assert np.array_equal(a, b)


def test_fused_sgd_update_matches_separate_update_kernel(monkeypatch):
    """One learner: the SGD update w' = w - lr g runs inside the weight-gradient GEMM epilogues
    (gradient never stored, shadow refreshed in place, GEMMs reordered so every weight's readers
    run before its update). Weights and losses over 3 steps (with an lr change) must equal the
    separate update kernel's bit for bit (ADPSGD_FUSED_UPDATE=1 vs default; opt-in)."""
    m = ModelDesc(layers=2, hidden=256, bidirectional=True, input_dim=260, proj=256, classes=1000, unroll=11)
    rng = np.random.default_rng(5)
    feats = rng.normal(size=(512, m.unroll, m.input_dim)).astype(np.float32)
    labels = rng.integers(0, m.classes, size=(512, m.unroll)).astype(np.int32)
    res = {}
    for off in ("1", "0"):
        monkeypatch.setenv("ADPSGD_FUSED_UPDATE", "0" if off == "1" else "1")
        g = LearnerGroup(m, StrategyConfig(learners=1, batch=256, seed=11), precision=Precision.BF16)
        g.set_dataset(feats, labels, 512)
        losses = [float(g.step(lr)[0]) for lr in (0.05, 0.05, 0.02)]
        res[off] = (losses, g.weights(0).copy())
        g.close()
    (l0, w0), (l1, w1) = res["0"], res["1"]
    assert l0 == l1
    assert np.array_equal(w0, w1)


def test_context_upload_is_stream_ordered():
    """Regression: w0 / the identity index / dataset uploads used pageable cudaMemcpy on the legacy
    stream, which the engine's non-blocking stream does not wait for (and which may return before
    the DMA lands): the bf16 shadow built right after could pick up the previous contents of the
    allocation. After a large context is freed, a new context's shadow must equal bf16(w0)."""
    import ctypes as C
    import torch
    from paper_2110_11199_b200 import _lib
    big = ModelDesc(layers=2, hidden=512, bidirectional=True, input_dim=260, proj=256, classes=4000, unroll=11)
    small = ModelDesc(layers=2, hidden=128, bidirectional=True, input_dim=40, proj=64, classes=96, unroll=7)
    for it in range(3):
        g = LearnerGroup(big, StrategyConfig(learners=1, batch=256, seed=it), precision=Precision.BF16)
        g.close()
        s = LearnerGroup(small, StrategyConfig(learners=1, batch=64, seed=4), precision=Precision.BF16)
        sh = np.zeros(s.D, dtype=np.uint16)
        _lib.check(_lib.lib().adpsgd_debug_buffer(s.handle, 102, sh.ctypes.data_as(C.c_void_p), sh.nbytes))
        ref = torch.from_numpy(s.weights(0).astype(np.float32)).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
        s.close()
        assert np.array_equal(sh, ref), it
