"""Cluster timing model and the coupled asynchronous run (proj/include/adpsgd/chronos.hpp).

ClusterProfile / effective_compute / simulate_wallclock / slowdown_experiment restate the
reference's scalar cost model (chronos.cpp:30-160) — the expected-ratio model of the straggler
study. coupled_run executes chronos::coupled_async (chronos.cpp:178-299) with the learners'
gradients, neighbour mixing and publications on the GPU (adpsgd_async_run), in the reference's
event order; its durations can come from the profile or from measured device step times.
"""
from __future__ import annotations

import ctypes as C
import heapq
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .engine import (LearnerGroup, ModelDesc, Precision, RunRecord, Strategy, StrategyConfig, iterations_per_epoch,
                     lr_at, run_training)
from .errors import ConfigError


@dataclass
class ClusterProfile:
    learners: int = 2
    compute_time: float = 1.0
    compute_multiplier: list = field(default_factory=list)
    comm_pairwise: float = 0.0
    comm_allreduce: float = 0.0
    sync_overhead: float = 0.0
    stragglers: list = field(default_factory=list)  # (learner_id, factor >= 1)

    def validate(self) -> None:  # chronos.cpp:30-49
        if self.learners < 1:
            raise ConfigError("cluster profile: learners must be >= 1")
        if self.compute_time <= 0.0:
            raise ConfigError("cluster profile: compute_time must be > 0")
        if self.comm_pairwise < 0 or self.comm_allreduce < 0 or self.sync_overhead < 0:
            raise ConfigError("cluster profile: communication times must be >= 0")
        if self.compute_multiplier and len(self.compute_multiplier) != self.learners:
            raise ConfigError("cluster profile: one compute multiplier per learner")
        if any(m <= 0 for m in self.compute_multiplier):
            raise ConfigError("cluster profile: multipliers must be > 0")
        for lid, f in self.stragglers:
            if lid < 0 or lid >= self.learners:
                raise ConfigError("cluster profile: straggler learner_id out of range")
            if f < 1.0:
                raise ConfigError("cluster profile: slowdown factor must be >= 1")

    def effective_compute(self, l: int) -> float:  # chronos.cpp:51-58
        c = self.compute_time
        if self.compute_multiplier:
            c *= self.compute_multiplier[l]
        for lid, f in self.stragglers:
            if lid == l:
                c *= f
        return c


def simulate_wallclock(strategy: Strategy, profile: ClusterProfile, iterations_per_learner: int) -> float:
    """Total simulated time of L * iterations batches (chronos.cpp:71-140)."""
    profile.validate()
    if iterations_per_learner < 1:
        raise ConfigError("iterations_per_learner must be >= 1")
    L = profile.learners
    if strategy in (Strategy.SDPSGD, Strategy.ADPSGD_D1D, Strategy.GENERIC):
        mx = max(profile.effective_compute(l) for l in range(L))
        if strategy != Strategy.SDPSGD:
            rnd = max(mx, profile.comm_allreduce) + profile.sync_overhead
        else:
            rnd = mx + profile.comm_allreduce + profile.sync_overhead
        return rnd * iterations_per_learner
    target = L * iterations_per_learner
    dur = [max(profile.effective_compute(l), profile.comm_pairwise) for l in range(L)]
    q = [(dur[l], l) for l in range(L)]
    heapq.heapify(q)
    t = 0.0
    for _ in range(target):
        t, l = heapq.heappop(q)
        heapq.heappush(q, (t + dur[l], l))
    return t


def slowdown_experiment(strategy: Strategy, base: ClusterProfile, factors, iterations_per_learner: int = 20):
    """Epoch-time ratio with learner 0 slowed by each factor (chronos.cpp:142-160)."""
    clean = ClusterProfile(base.learners, base.compute_time, list(base.compute_multiplier), base.comm_pairwise,
                           base.comm_allreduce, base.sync_overhead, [])
    t0 = simulate_wallclock(strategy, clean, iterations_per_learner)
    out = []
    for f in factors:
        if f < 1.0:
            raise ConfigError("slowdown factors must be >= 1")
        slow = ClusterProfile(clean.learners, clean.compute_time, list(clean.compute_multiplier), clean.comm_pairwise,
                              clean.comm_allreduce, clean.sync_overhead, [(0, f)])
        t1 = simulate_wallclock(strategy, slow, iterations_per_learner)
        out.append({"factor": f, "baseline_epoch_time": t0, "straggler_epoch_time": t1, "ratio": t1 / t0})
    return out


def async_run(group: LearnerGroup, strategy: Strategy, durations, target: int, ipe: int, lr_per_epoch):
    d = np.ascontiguousarray(durations, dtype=np.float64)
    lrs = np.ascontiguousarray(lr_per_epoch, dtype=np.float64)
    ev = np.zeros(target, dtype=np.int32)
    et = np.zeros(target, dtype=np.float64)
    n = C.c_int64()
    _lib.check(_lib.lib().adpsgd_async_run(group.handle, int(strategy), d.ctypes.data_as(C.POINTER(C.c_double)),
                                           target, ipe, lrs.ctypes.data_as(C.POINTER(C.c_double)), len(lrs),
                                           ev.ctypes.data_as(C.POINTER(C.c_int32)),
                                           et.ctypes.data_as(C.POINTER(C.c_double)), C.byref(n)))
    return ev[:n.value], et[:n.value]


def coupled_run(profile: ClusterProfile, cfg: StrategyConfig, group: LearnerGroup, train_count: int):
    """chronos::coupled_run (chronos.cpp:303-321) for FM/RM: cfg.epochs x ipe x L updates in the
    coupled event order on the device. Returns (event learners, event times, total time)."""
    profile.validate()
    cfg.validate()
    if profile.learners != cfg.learners:
        raise ConfigError("cluster profile learner count does not match strategy config")
    if cfg.strategy not in (Strategy.ADPSGD_FM, Strategy.ADPSGD_RM):
        raise ConfigError("coupled async runs FM or RM (synchronous strategies use run_training)")
    ipe = iterations_per_epoch(cfg, train_count)
    dur = [max(profile.effective_compute(l), profile.comm_pairwise) for l in range(cfg.learners)]
    target = cfg.epochs * ipe * cfg.learners
    # lr of a learner's own round r is lr_at(cfg.lr, r / ipe) (chronos.cpp:216); a fast learner can
    # run up to `target` rounds, past cfg.epochs epochs, so the table covers every reachable epoch
    lrs = [lr_at(cfg.lr, e) for e in range((target - 1) // ipe + 1)]
    ev, et = async_run(group, cfg.strategy, dur, target, ipe, lrs)
    return ev, et, float(et[-1]) if len(et) else 0.0


@dataclass
class CoupledResult:
    record: RunRecord
    total_time: float


def coupled_training(profile: ClusterProfile, cfg: StrategyConfig, model: ModelDesc, feats, labels,
                     train_count: int, precision: Precision = Precision.BF16, device: int = 0,
                     synth: tuple | None = None) -> CoupledResult:
    """chronos::coupled_run (chronos.cpp:303-321) with its RunRecord. FM/RM: the coupled
    asynchronous replay on the device with the record of chronos.cpp:271-289 (consensus after
    every L updates, per-epoch held-out / train loss of the averaged model, divergence stop);
    synchronous strategies: run_training for the record and the cost model for the clock.
    synth = (n_seg, seed) selects the device-generated dataset when feats is None."""
    profile.validate()
    cfg.validate()
    if profile.learners != cfg.learners:
        raise ConfigError("cluster profile learner count does not match strategy config")
    ipe = iterations_per_epoch(cfg, train_count)
    if cfg.strategy not in (Strategy.ADPSGD_FM, Strategy.ADPSGD_RM):
        rec = run_training(cfg, model, feats, labels, train_count, precision=precision, device=device, synth=synth)
        return CoupledResult(rec, simulate_wallclock(cfg.strategy, profile, ipe * cfg.epochs))
    g = LearnerGroup(model, cfg, precision=precision, device=device)
    try:
        if feats is None:
            n_seg, seed = synth
            g.synth_dataset(n_seg, train_count, seed)
        else:
            g.set_dataset(feats, labels, train_count)
            n_seg = np.asarray(feats).shape[0]
        L = cfg.learners
        held = np.arange(train_count, n_seg, dtype=np.int32)
        train = np.arange(train_count, dtype=np.int32)
        initial = g.eval_loss(g.averaged_model(), held) if len(held) else float("nan")
        dur = np.ascontiguousarray([max(profile.effective_compute(l), profile.comm_pairwise) for l in range(L)],
                                   dtype=np.float64)
        target = cfg.epochs * ipe * L
        lrs = np.ascontiguousarray([lr_at(cfg.lr, e) for e in range((target - 1) // ipe + 1)], dtype=np.float64)
        cons = np.zeros(cfg.epochs * ipe, dtype=np.float64)
        hl = np.zeros(cfg.epochs, dtype=np.float64)
        tl = np.zeros(cfg.epochs, dtype=np.float64)
        et = np.zeros(target, dtype=np.float64)
        dp = C.POINTER(C.c_double)
        ip = C.POINTER(C.c_int32)
        r = _lib.AsyncRecord()
        r.heldout_idx, r.n_heldout = held.ctypes.data_as(ip), len(held)
        r.train_idx, r.n_train = train.ctypes.data_as(ip), len(train)
        r.initial_heldout = initial
        r.consensus, r.cap_iters = cons.ctypes.data_as(dp), len(cons)
        r.heldout, r.train, r.cap_epochs = hl.ctypes.data_as(dp), tl.ctypes.data_as(dp), cfg.epochs
        n = C.c_int64()
        _lib.check(_lib.lib().adpsgd_async_run_record(g.handle, int(cfg.strategy), dur.ctypes.data_as(dp), target, ipe,
                                                      lrs.ctypes.data_as(dp), len(lrs), None, et.ctypes.data_as(dp),
                                                      C.byref(r), C.byref(n)))
        rec = RunRecord()
        rec.iterations = [(k, float(cons[k]), lr_at(cfg.lr, k // ipe)) for k in range(r.n_iters)]
        rec.epochs = [(e, float(hl[e]), float(tl[e]), lr_at(cfg.lr, e)) for e in range(r.n_epochs)]
        rec.diverged = r.diverged_epoch >= 0
        rec.divergence_epoch = r.diverged_epoch
        rec.iteration_count = len(rec.iterations)
        rec.final_model = g.averaged_model()
        return CoupledResult(rec, float(et[n.value - 1]) if n.value else 0.0)
    finally:
        g.close()
