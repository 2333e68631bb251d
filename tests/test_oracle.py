"""Pin the CPU oracle before trusting it (CPU only).

* pairing / RNG against tests/golden/pairing.json, produced from the reference's own
  rng.hpp (oracle/_ref) — bit-exact;
* LSTM loss/gradient against torch fp64 fixtures and central finite differences
  (proj/src/verify.cpp:25-59 pattern);
* engine steps against the reference's own algebraic tests
  (proj/tests/test_engine.cpp:96-342, test_mixing.cpp:19-138).
"""
import hashlib
import json
import os
from collections import Counter

import numpy as np
import pytest

GOLD = os.path.join(os.path.dirname(__file__), "golden")
S_SDPSGD, S_FM, S_RM, S_D1D, S_GENERIC = range(5)
MIX_FIXED, MIX_RANDOM, MIX_UNIFORM = range(3)


@pytest.fixture(scope="module")
def pairing():
    with open(os.path.join(GOLD, "pairing.json")) as f:
        return json.load(f)


def test_pairing_short_golden(oracle_mod, pairing):
    O = oracle_mod
    for key, seqs in pairing["short"].items():
        s, L = map(int, key.split("/"))
        for k, want in enumerate(seqs):
            assert O.permutation_for_iteration(s, L, k).tolist() == want, (key, k)


def test_pairing_long_golden(oracle_mod, pairing):
    O = oracle_mod
    for key, digest in pairing["long_sha256"].items():
        s, L = map(int, key.split("/"))
        h = hashlib.sha256()
        for k in range(10000):
            h.update(O.permutation_for_iteration(s, L, k).tobytes())
        assert h.hexdigest() == digest, key


def test_survey_appendix_a_vectors(oracle_mod):
    # SURVEY.md Appendix A (generated from rng.hpp).
    O = oracle_mod
    assert O.permutation_for_iteration(0, 8, 0).tolist() == [4, 0, 2, 1, 6, 7, 3, 5]
    assert O.permutation_for_iteration(2025, 8, 3).tolist() == [2, 4, 7, 3, 0, 5, 1, 6]
    lib = O.lib()
    assert lib.or_derive_seed(0, 0xC001) == 6450415292512655039
    assert lib.or_derive_seed3(0, 0xC001, 0) == 3295359393989930592
    assert lib.or_derive_seed(1234, 0xA001) == 6855522026284859676
    assert lib.or_derive_seed(1234, 0xB003) == 9831948877771049344
    assert lib.or_mt_first(42) == 13930160852258120406
    # Learner 4 sits at ring position 0: left 5, right 0 (Appendix A example).
    assert O.ring_neighbors(S_RM, 0, 8, 0, 4) == (5, 0)
    assert O.ring_neighbors(S_RM, 0, 8, 0, 0) == (4, 2)


def test_w0_and_batches_golden(oracle_mod, pairing):
    O = oracle_mod
    w0 = O.init_w0(1234, 16)
    assert [float.hex(float(x)) for x in w0] == pairing["w0"]["1234"]
    for key, want in pairing["batches"].items():
        s, l, _, _ = key.split("/")
        got = O.learner_batches(int(s), int(l), 5, 8, 1000)
        assert got.tolist() == want


def test_permutation_chi_square(oracle_mod):
    # test_mixing.cpp:72-87 analogue on the per-iteration streams.
    O = oracle_mod
    counts = Counter(tuple(O.permutation_for_iteration(2024, 4, k)) for k in range(24000))
    assert len(counts) == 24
    exp = 24000 / 24
    chi2 = sum((n - exp) ** 2 / exp for n in counts.values())
    assert chi2 < 49.7


def test_ring_matrices(oracle_mod):
    O = oracle_mod
    third = 1.0 / 3.0
    m3 = O.mixing_matrix(MIX_FIXED, 3)
    assert np.allclose(m3, third, atol=1e-15)
    m5 = O.mixing_matrix(MIX_FIXED, 5)
    assert m5[0].tolist() == [third, third, 0.0, 0.0, third]
    with pytest.raises(ValueError):
        O.mixing_matrix(MIX_FIXED, 2)
    import itertools
    for p in itertools.permutations(range(5)):
        m = O.mixing_matrix(MIX_RANDOM, 5, p)
        assert np.allclose(m.sum(0), 1) and np.allclose(m.sum(1), 1)
        assert set(np.unique(m)) <= {0.0, third}
    # RM neighbours agree with the dense random ring's nonzero pattern.
    for k in range(20):
        perm = O.permutation_for_iteration(99, 7, k)
        T = O.mixing_matrix(MIX_RANDOM, 7, perm)
        for l in range(7):
            left, right = O.ring_neighbors(S_RM, 99, 7, k, l)
            assert sorted(np.nonzero(T[:, l])[0].tolist()) == sorted({l, left, right})


def test_lr_schedule(oracle_mod):
    # test_engine.cpp:32-47
    f = oracle_mod.lib().or_lr_at
    assert f(0.32, 3.2, 10, 0.7071067811865476, 1 << 30, 0) == pytest.approx(0.32, rel=1e-15)
    assert f(0.32, 3.2, 10, 0.7071067811865476, 1 << 30, 5) == pytest.approx(0.32 + 2.88 * 0.5, rel=1e-12)
    assert f(0.32, 3.2, 10, 0.7071067811865476, 12, 14) == pytest.approx(1.6, rel=1e-12)


@pytest.mark.parametrize("name", ["uni2", "bi2p", "bi3p_t21"])
def test_lstm_vs_torch_golden(oracle_mod, name):
    O = oracle_mod
    z = np.load(os.path.join(GOLD, f"lstm_{name}.npz"))
    d = O.desc(*[int(x) for x in z["case"][:7]])
    loss, g = O.lstm_loss_grad(d, z["w"], z["feats"], z["labels"], z["idx"])
    assert abs(loss - float(z["loss"])) <= 1e-12
    assert np.max(np.abs(g - z["grad"])) <= 1e-12


def test_lstm_finite_differences(oracle_mod):
    # verify.cpp:25-59: central differences, h = 1e-5, rel err vs max(1, |g|).
    O = oracle_mod
    d = O.desc(2, 5, 1, 4, 3, 6, 6)
    D = O.param_count(d)
    rng = np.random.default_rng(5)
    w = rng.normal(0, 0.4, D)
    feats = rng.normal(size=(4, 6, 4)).astype(np.float32)
    labels = rng.integers(0, 6, size=(4, 6)).astype(np.int32)
    idx = np.array([0, 3, 1], dtype=np.int32)
    _, g = O.lstm_loss_grad(d, w, feats, labels, idx)
    h = 1e-5
    for p in rng.choice(D, 40, replace=False):
        wp, wm = w.copy(), w.copy()
        wp[p] += h
        wm[p] -= h
        fd = (O.lstm_loss_grad(d, wp, feats, labels, idx, want_grad=False)
              - O.lstm_loss_grad(d, wm, feats, labels, idx, want_grad=False)) / (2 * h)
        assert abs(fd - g[p]) / max(1.0, abs(g[p])) <= 1e-6


def test_lstm_threads_deterministic(oracle_mod):
    O = oracle_mod
    z = np.load(os.path.join(GOLD, "lstm_bi2p.npz"))
    d = O.desc(*[int(x) for x in z["case"][:7]])
    idx = np.arange(6, dtype=np.int32)
    l1, g1 = O.lstm_loss_grad(d, z["w"], z["feats"], z["labels"], idx, threads=1)
    l3, g3 = O.lstm_loss_grad(d, z["w"], z["feats"], z["labels"], idx, threads=3)
    assert abs(l1 - l3) < 1e-13 and np.max(np.abs(g1 - g3)) < 1e-15


# ---- engine algebra (reference test_engine.cpp) ---------------------------

def _tiny(O, L=5, M=3, seed=13, depth=2):
    d = O.desc(1, 4, 0, 3, 0, 5, 4)
    rng = np.random.default_rng(seed)
    feats = rng.normal(size=(32, 4, 3)).astype(np.float32)
    labels = rng.integers(0, 5, size=(32, 4)).astype(np.int32)
    return O.OracleEngine(d, L, M, seed, feats, labels, 28, history_depth=depth), d, feats, labels


def test_sdpsgd_equals_pooled_sgd(oracle_mod):
    # test_engine.cpp:111-125
    O = oracle_mod
    e, d, feats, labels = _tiny(O, L=4, M=5, seed=11)
    w0 = e.model(0)
    pooled = np.concatenate([O.learner_batches(11, l, 1, 5, 28)[0] for l in range(4)])
    _, g = O.lstm_loss_grad(d, w0, feats, labels, pooled)
    assert e.step(S_SDPSGD, 0.05, 0) == 0
    for l in range(4):
        assert np.max(np.abs(e.model(l) - (w0 - 0.05 * g))) <= 1e-10
    w = e.model(1)
    w[0] += 1e-6
    e.set_model(1, w)
    assert e.step(S_SDPSGD, 0.05, 1) == 5  # SyncViolationError


def test_mixing_step_dense_oracle(oracle_mod):
    # test_engine.cpp:127-147
    O = oracle_mod
    e, d, feats, labels = _tiny(O)
    assert e.step(S_D1D, 0.1, 0) == 0
    W = np.stack([e.model(l) for l in range(5)], 1)
    G = np.zeros_like(W)
    for l in range(5):
        idx = O.learner_batches(13, l, 2, 3, 28)[1]
        G[:, l] = O.lstm_loss_grad(d, W[:, l], feats, labels, idx)[1]
    expected = W @ O.mixing_matrix(MIX_FIXED, 5) - 0.07 * G
    assert e.step(S_FM, 0.07, 1) == 0
    got = np.stack([e.model(l) for l in range(5)], 1)
    assert np.max(np.abs(got - expected)) <= 1e-14


def test_mixing_preserves_mean_and_d1d_consensus(oracle_mod):
    # test_engine.cpp:149-161, 180-215
    O = oracle_mod
    for strat in (S_FM, S_RM):
        e, *_ = _tiny(O, seed=17)
        e.step(S_D1D, 0.2, 0)
        mean = np.mean([e.model(l) for l in range(5)], 0)
        e.step(strat, 0.0, 1)
        assert np.max(np.abs(np.mean([e.model(l) for l in range(5)], 0) - mean)) <= 1e-12
    e, *_ = _tiny(O, L=4, seed=23)
    e.step(S_D1D, 0.1, 0)
    mean = np.mean([e.model(l) for l in range(4)], 0)
    e.step(S_D1D, 0.0, 1)
    for l in range(4):
        assert np.max(np.abs(e.model(l) - mean)) <= 1e-15


def test_generic_tau0_equals_mixing_and_d1d(oracle_mod):
    # test_engine.cpp:236-294
    O = oracle_mod
    a, *_ = _tiny(O, seed=31, depth=3)
    b, *_ = _tiny(O, seed=31, depth=3)
    for k in range(3):
        a.step(S_FM, 0.05, k)
        b.step(S_GENERIC, 0.05, k, generic_mix=MIX_FIXED, taus=[0] * 5)
    assert max(np.max(np.abs(a.model(l) - b.model(l))) for l in range(5)) == 0.0
    a, *_ = _tiny(O, L=4, seed=37, depth=3)
    b, *_ = _tiny(O, L=4, seed=37, depth=3)
    for k in range(3):
        a.step(S_D1D, 0.05, k)
        b.step(S_GENERIC, 0.05, k, generic_mix=MIX_UNIFORM, taus=[0] * 4)
        assert max(np.max(np.abs(a.model(l) - b.model(l))) for l in range(4)) <= 1e-14
    c, *_ = _tiny(O, L=3, seed=43, depth=2)
    assert c.step(S_GENERIC, 0.05, 0, generic_mix=MIX_UNIFORM, taus=[0, 2, 0]) == 6


def test_single_learner_is_sgd_for_every_strategy(oracle_mod):
    # test_engine.cpp:321-342
    O = oracle_mod
    ref, *_ = _tiny(O, L=1, seed=99)
    for k in range(3):
        ref.step(S_SDPSGD, 0.05, k)
    for s in (S_FM, S_RM, S_D1D, S_GENERIC):
        e, *_ = _tiny(O, L=1, seed=99)
        for k in range(3):
            assert e.step(s, 0.05, k) == 0
        assert np.array_equal(e.model(0), ref.model(0))


def test_fm_rm_reject_two_learners(oracle_mod):
    # engine.cpp:62-65
    O = oracle_mod
    e, *_ = _tiny(O, L=2)
    assert e.step(S_FM, 0.1, 0) == 8
    assert e.step(S_RM, 0.1, 0) == 8
    assert e.step(S_D1D, 0.1, 0) == 0


def test_injected_step_matches_formula(oracle_mod):
    O = oracle_mod
    e, *_ = _tiny(O, L=6, seed=3)
    e.step(S_D1D, 0.3, 0)
    D = e.D
    rng = np.random.default_rng(0)
    G = rng.normal(size=(6, D))
    W = np.stack([e.model(l) for l in range(6)])
    assert e.step_injected(S_RM, 0.1, 5, G) == 0
    for l in range(6):
        left, right = O.ring_neighbors(S_RM, 3, 6, 5, l)
        want = (W[l] + W[left] + W[right]) / 3.0 - 0.1 * G[l]
        assert np.max(np.abs(e.model(l) - want)) <= 1e-15
