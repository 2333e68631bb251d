"""CPU-only checks of the C-ABI library: it loads, exports every symbol the header
declares, and its pure-host entry points (pairing, parameter layout, lr schedule,
config validation) are bit-exact with the reference / oracle. No kernel runs here."""
import ctypes as C
import json
import os

import numpy as np
import pytest

from paper_2110_11199_b200 import _lib
from paper_2110_11199_b200 import engine as E
from paper_2110_11199_b200.errors import ConfigError, InvalidOrderError

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def test_library_exports_header_symbols():
    L = _lib.lib()
    syms = _lib.header_symbols()
    assert len(syms) >= 30
    for s in syms:
        assert hasattr(L, s), s
    assert b"sm_100a" in L.adpsgd_build_info()


def test_pairing_bit_exact_with_reference_golden():
    with open(os.path.join(GOLD, "pairing.json")) as f:
        fx = json.load(f)
    for key, seqs in fx["short"].items():
        s, L = map(int, key.split("/"))
        for k, want in enumerate(seqs):
            assert E.permutation_for_iteration(s, L, k) == want


def test_pairing_long_sequences_match_oracle(oracle_mod):
    for L in (3, 5, 8, 16, 64):
        for k in range(0, 10000, 97):
            assert E.permutation_for_iteration(1234, L, k) == oracle_mod.permutation_for_iteration(1234, L, k).tolist()


def test_neighbours_match_oracle(oracle_mod):
    for strat in (E.Strategy.ADPSGD_FM, E.Strategy.ADPSGD_RM):
        for L in (3, 4, 8, 13):
            for k in range(30):
                _, lr = E.pairing(strat, 2025, L, k)
                for l in range(L):
                    assert lr[l] == oracle_mod.ring_neighbors(int(strat), 2025, L, k, l)
    with pytest.raises(InvalidOrderError):
        E.pairing(E.Strategy.ADPSGD_FM, 0, 2, 0)


def test_param_count_matches_oracle(oracle_mod):
    for args in [(2, 256, 0, 40, 0, 32, 21), (6, 512, 1, 260, 256, 32000, 21), (6, 1024, 1, 260, 256, 32000, 21),
                 (3, 16, 1, 12, 8, 11, 21)]:
        m = E.ModelDesc(*args)
        assert m.param_count() == oracle_mod.param_count(oracle_mod.desc(*args))
    assert E.ModelDesc().param_count() == 145145344
    assert E.ModelDesc(hidden=512).param_count() == 43130368
    assert E.ModelDesc(hidden=512).train_flops_per_frame() == 256311296
    assert E.ModelDesc().train_flops_per_frame() == 866123776


def test_lr_schedule_matches_reference():
    s = E.LrSchedule(base_lr=0.32, peak_lr=3.2, warmup_epochs=10)
    assert E.lr_at(s, 0) == pytest.approx(0.32, rel=1e-15)
    assert E.lr_at(s, 5) == pytest.approx(0.32 + (3.2 - 0.32) * 0.5, rel=1e-12)
    assert E.lr_at(s, 20) == pytest.approx(3.2, rel=1e-15)
    s.anneal_start_epoch = 12
    assert E.lr_at(s, 14) == pytest.approx(1.6, rel=1e-12)


def test_strategy_names_round_trip():
    for s in E.Strategy:
        assert E.strategy_from_name(E.strategy_name(s)) == s
    with pytest.raises(ConfigError):
        E.strategy_from_name("BMUF")


def test_config_validation_without_gpu():
    # engine.cpp:60-77 — rejected before any device work
    cfg = E.StrategyConfig(strategy=E.Strategy.ADPSGD_FM, learners=2)
    with pytest.raises(ConfigError):
        cfg.validate()
    c = _lib.Config()
    c.model = E.ModelDesc(2, 16, True, 8, 8, 16, 4).c()
    c.strategy, c.learners, c.local_learners, c.batch = 1, 2, 2, 4
    h = C.c_void_p()
    rc = _lib.lib().adpsgd_ctx_create(C.byref(c), C.byref(h))
    assert rc == ConfigError.code
    assert "at least 3 learners" in _lib.last_error()
    c.strategy, c.learners, c.batch = 3, 2, 0
    assert _lib.lib().adpsgd_ctx_create(C.byref(c), C.byref(h)) == ConfigError.code
    c.batch, c.precision = 4, 1
    c.model = E.ModelDesc(2, 12, True, 8, 8, 16, 4).c()  # hidden not a multiple of 8 in bf16 mode
    assert _lib.lib().adpsgd_ctx_create(C.byref(c), C.byref(h)) == ConfigError.code


def test_csv_format_and_ipe():
    from paper_2110_11199_b200.engine import RunRecord, fmt_double, iterations_per_epoch, write_csv
    import tempfile, os
    assert fmt_double(0.1) == "0.10000000000000001"
    assert iterations_per_epoch(E.StrategyConfig(learners=8, batch=1024), 65536) == 8
    assert iterations_per_epoch(E.StrategyConfig(learners=4, batch=64), 100) == 1
    r = RunRecord(iterations=[(0, 0.5, 0.1)], epochs=[(0, 2.5, 2.25, 0.1)])
    with tempfile.TemporaryDirectory() as d:
        write_csv(r, d)
        assert open(os.path.join(d, "consensus.csv")).read().splitlines() == ["k,distance", "0,0.5"]
        assert open(os.path.join(d, "run.csv")).read().splitlines() == ["epoch,heldout_loss,lr",
                                                                          "0,2.5,0.10000000000000001"]
        write_csv(r, d, stem="ADPSGD_FM_f5_")
        assert os.path.exists(os.path.join(d, "ADPSGD_FM_f5_run.csv"))


def test_wallclock_model_matches_reference_known_answers():
    # test_chronos.cpp:47-76, 110-129
    from paper_2110_11199_b200 import chronos as CH
    from paper_2110_11199_b200.engine import Strategy as S
    h = lambda L, **kw: CH.ClusterProfile(learners=L, compute_time=1.0, comm_pairwise=0.01, comm_allreduce=0.1, **kw)
    assert CH.simulate_wallclock(S.SDPSGD, h(4), 10) == pytest.approx(11.0, rel=1e-12)
    assert CH.simulate_wallclock(S.ADPSGD_D1D, h(4), 10) == pytest.approx(10.0, rel=1e-12)
    assert CH.simulate_wallclock(S.SDPSGD, h(4, sync_overhead=0.05), 10) == pytest.approx(11.5, rel=1e-12)
    assert CH.simulate_wallclock(S.ADPSGD_FM, h(4), 10) == pytest.approx(10.0, rel=1e-12)
    slow = CH.simulate_wallclock(S.ADPSGD_FM, h(16, stragglers=[(0, 100.0)]), 20)
    assert slow / CH.simulate_wallclock(S.ADPSGD_FM, h(16), 20) <= 16.0 / 15.0 + 0.1
    rep = CH.slowdown_experiment(S.ADPSGD_D1D, h(16), [1.0, 5.0, 10.0, 100.0], 20)
    assert rep[0]["ratio"] == pytest.approx(1.0) and rep[3]["ratio"] == pytest.approx(100.0, rel=0.05)
    assert CH.slowdown_experiment(S.ADPSGD_FM, h(16), [100.0], 20)[0]["ratio"] <= 2.0
    with pytest.raises(ConfigError):
        CH.slowdown_experiment(S.ADPSGD_FM, h(16), [0.5], 20)


def test_consensus_from_gram_matches_numpy():
    """adpsgd_consensus_from_gram (host Jacobi) = sqrt(lambda_max) as SelfAdjointEigenSolver gives
    it (mixing.cpp:174-179); pure host code, no GPU."""
    from paper_2110_11199_b200.engine import consensus_from_gram
    rng = np.random.default_rng(5)
    for L in (2, 3, 8, 16):
        X = rng.normal(size=(L, 40))
        X -= X.mean(axis=0)
        G = X @ X.T
        want = np.sqrt(np.linalg.eigvalsh(G).max())
        assert abs(consensus_from_gram(G) - want) <= 1e-10 * want
