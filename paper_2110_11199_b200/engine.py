"""Host-side mirror of the reference learner API (proj/include/adpsgd/engine.hpp), backed by
the B200 C ABI. Same names, argument meaning and error behaviour as the reference:

  Strategy / strategy_name / strategy_from_name      engine.hpp:17-20, engine.cpp:25-43
  LrSchedule / lr_at                                 engine.hpp:25-33, engine.cpp:45-58
  StrategyConfig.validate                            engine.hpp:35-50, engine.cpp:60-77
  permutation_for_iteration                          engine.hpp:85-86, engine.cpp:130-134
  LearnerGroup.step (step_sdpsgd / step_adpsgd_mixing / step_d1d / step_generic_staleness)
                                                     engine.hpp:88-105, engine.cpp:136-204
  LstmObjective (Objective plugin)                   objectives.hpp:45-69

The learners' models, gradients and activations live on the GPU; only O(M) sampling
indices and the pairing (O(L)) are produced on the host, bit-exactly as the reference does.
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .errors import ConfigError, InvalidStateError


class Strategy(enum.IntEnum):
    SDPSGD = 0
    ADPSGD_FM = 1
    ADPSGD_RM = 2
    ADPSGD_D1D = 3
    GENERIC = 4


class MixKind(enum.IntEnum):
    FIXED_RING = 0
    RANDOM_RING = 1
    UNIFORM = 2


class AsyncMode(enum.IntEnum):
    """adpsgd_async_mode: FREE reads neighbours' latest publications (never waits); LOCKSTEP reads
    exactly version k (== synchronous FM/RM); BOUNDED waits until the latest is >= k - max_lag."""
    FREE = 0
    LOCKSTEP = 1
    BOUNDED = 2


class Precision(enum.IntEnum):
    FP32 = 0
    BF16 = 1


_NAMES = {Strategy.SDPSGD: "SDPSGD", Strategy.ADPSGD_FM: "ADPSGD_FM", Strategy.ADPSGD_RM: "ADPSGD_RM",
          Strategy.ADPSGD_D1D: "ADPSGD_D1D", Strategy.GENERIC: "GENERIC"}


def strategy_name(s: Strategy) -> str:
    return _NAMES.get(Strategy(s), "unknown")


def strategy_from_name(name: str) -> Strategy:
    for s, n in _NAMES.items():
        if n == name:
            return s
    raise ConfigError("unknown strategy: " + name)


@dataclass
class LrSchedule:
    base_lr: float = 0.1
    peak_lr: float = 0.1
    warmup_epochs: int = 0
    anneal_factor: float = 0.7071067811865476
    anneal_start_epoch: int = 1 << 30


def lr_at(s: LrSchedule, epoch: int) -> float:
    if epoch < 0:
        raise InvalidStateError("lr_at: epoch must be >= 0")
    return float(_lib.lib().adpsgd_lr_at(s.base_lr, s.peak_lr, s.warmup_epochs, s.anneal_factor,
                                         s.anneal_start_epoch, epoch))


@dataclass
class ModelDesc:
    """BLSTM acoustic model. hidden = cells per direction."""
    layers: int = 6
    hidden: int = 1024
    bidirectional: bool = True
    input_dim: int = 260
    proj: int = 256
    classes: int = 32000
    unroll: int = 21

    def c(self) -> _lib.ModelDesc:
        return _lib.ModelDesc(self.layers, self.hidden, int(self.bidirectional), self.input_dim, self.proj,
                              self.classes, self.unroll)

    def param_count(self) -> int:
        return int(_lib.lib().adpsgd_param_count(C.byref(self.c())))

    def fwd_flops_per_frame(self) -> float:
        nd = 2 if self.bidirectional else 1
        f = 0.0
        for l in range(self.layers):
            i = self.input_dim if l == 0 else nd * self.hidden
            f += 2.0 * nd * 4 * self.hidden * (i + self.hidden)
        top = nd * self.hidden
        if self.proj > 0:
            f += 2.0 * top * self.proj
        f += 2.0 * (self.proj if self.proj > 0 else top) * self.classes
        return f

    def train_flops_per_frame(self) -> float:
        nd = 2 if self.bidirectional else 1
        return 3.0 * self.fwd_flops_per_frame() - 2.0 * nd * 4 * self.hidden * self.input_dim

    def param_blocks(self) -> list:
        """(name, slice, fan_in) of every parameter block of the flat vector, in layout order
        (csrc/model.hpp: per layer, per direction W_ih, W_hh, b; then W_proj, b_proj, W_out, b_out)."""
        nd = 2 if self.bidirectional else 1
        H, off, out = self.hidden, 0, []

        def add(name, n, fan_in):
            nonlocal off
            out.append((name, slice(off, off + n), fan_in))
            off += n

        for l in range(self.layers):
            i = self.input_dim if l == 0 else nd * H
            for d in range(nd):
                add(f"l{l}d{d}.w_ih", 4 * H * i, i)
                add(f"l{l}d{d}.w_hh", 4 * H * H, H)
                add(f"l{l}d{d}.b", 4 * H, H)
        top = nd * H
        if self.proj > 0:
            add("w_proj", self.proj * top, top)
            add("b_proj", self.proj, top)
        oi = self.proj if self.proj > 0 else top
        add("w_out", self.classes * oi, oi)
        add("b_out", self.classes, oi)
        return out


@dataclass
class StrategyConfig:
    strategy: Strategy = Strategy.SDPSGD
    learners: int = 2
    batch: int = 1
    epochs: int = 1
    lr: LrSchedule = field(default_factory=LrSchedule)
    seed: int = 0
    staleness_cap: int = 1
    staleness: list = field(default_factory=list)
    generic_mix: MixKind = MixKind.UNIFORM

    def validate(self) -> None:  # engine.cpp:60-77
        if self.learners < 1:
            raise ConfigError("learners must be >= 1")
        if self.strategy in (Strategy.ADPSGD_FM, Strategy.ADPSGD_RM) and self.learners != 1 and self.learners < 3:
            raise ConfigError("FM/RM mixing requires at least 3 learners")
        if self.batch < 1:
            raise ConfigError("batch must be >= 1")
        if self.epochs < 1:
            raise ConfigError("epochs must be >= 1")
        if self.staleness_cap < 0:
            raise ConfigError("staleness_cap must be >= 0")
        if self.staleness and len(self.staleness) != self.learners:
            raise ConfigError("staleness list must have one entry per learner")
        for tau in self.staleness:
            if tau < 0 or tau > self.staleness_cap:
                raise ConfigError("staleness entries must lie in [0, staleness_cap]")


def permutation_for_iteration(seed: int, learners: int, iteration: int) -> list:
    out = (C.c_int32 * learners)()
    _lib.check(_lib.lib().adpsgd_permutation_for_iteration(seed, learners, iteration, out))
    return list(out)


def pairing(strategy: Strategy, seed: int, learners: int, iteration: int):
    """(mapping, [(left, right) per learner]) for FM or RM at iteration k (chronos.cpp:224-235)."""
    m = (C.c_int32 * learners)()
    lr = (C.c_int32 * (2 * learners))()
    _lib.check(_lib.lib().adpsgd_pairing(int(strategy), seed, learners, iteration, m, lr))
    return list(m), [(lr[2 * i], lr[2 * i + 1]) for i in range(learners)]


def _ptr(a: np.ndarray, ct):
    return a.ctypes.data_as(C.POINTER(ct))


class LearnerGroup:
    """The vector<LearnerState> of engine::run_training, device-resident: `local_learners`
    learners of a global ring of `cfg.learners`, hosted on one GPU."""

    def __init__(self, model: ModelDesc, cfg: StrategyConfig, precision: Precision = Precision.BF16, device: int = 0,
                 first_learner: int = 0, local_learners: int | None = None):
        cfg.validate()
        self.model, self.cfg, self.precision = model, cfg, Precision(precision)
        self.local = cfg.learners if local_learners is None else local_learners
        self.first = first_learner
        c = _lib.Config()
        c.model = model.c()
        c.precision = int(precision)
        c.strategy = int(cfg.strategy)
        c.learners = cfg.learners
        c.first_learner = first_learner
        c.local_learners = self.local
        c.batch = cfg.batch
        c.device = device
        c.generic_mix = int(cfg.generic_mix)
        c.staleness_cap = cfg.staleness_cap
        c.seed = cfg.seed
        h = C.c_void_p()
        _lib.check(_lib.lib().adpsgd_ctx_create(C.byref(c), C.byref(h)))
        self._h = h
        self.D = model.param_count()

    def close(self) -> None:
        if getattr(self, "_h", None):
            _lib.lib().adpsgd_ctx_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def handle(self):
        return self._h

    # ---- data ----
    def set_dataset(self, feats: np.ndarray, labels: np.ndarray, train_count: int) -> None:
        feats = np.ascontiguousarray(feats, dtype=np.float32)
        labels = np.ascontiguousarray(labels, dtype=np.int32)
        _lib.check(_lib.lib().adpsgd_set_dataset(self._h, _ptr(feats, C.c_float), _ptr(labels, C.c_int32),
                                                 feats.shape[0], train_count))
        self.n_seg = feats.shape[0]

    def synth_dataset(self, n_seg: int, train_count: int, seed: int) -> None:
        _lib.check(_lib.lib().adpsgd_synth_dataset(self._h, n_seg, train_count, seed))
        self.n_seg = n_seg

    def dataset(self):
        m = self.model
        f = np.zeros((self.n_seg, m.unroll, m.input_dim), dtype=np.float32)
        l = np.zeros((self.n_seg, m.unroll), dtype=np.int32)
        _lib.check(_lib.lib().adpsgd_get_dataset(self._h, _ptr(f, C.c_float), _ptr(l, C.c_int32)))
        return f, l

    # ---- models ----
    def weights(self, j: int) -> np.ndarray:
        w = np.zeros(self.D, dtype=np.float64)
        _lib.check(_lib.lib().adpsgd_get_weights(self._h, j, _ptr(w, C.c_double), self.D))
        return w

    def set_weights(self, j: int, w) -> None:
        w = np.ascontiguousarray(w, dtype=np.float64)
        _lib.check(_lib.lib().adpsgd_set_weights(self._h, j, _ptr(w, C.c_double), self.D))

    @property
    def iteration(self) -> int:
        return int(_lib.lib().adpsgd_iteration(self._h))

    # ---- steps ----
    def _taus(self, taus):
        if taus is None:
            return None, None
        t = np.ascontiguousarray(taus, dtype=np.int32)
        return t, _ptr(t, C.c_int32)

    def step(self, lr: float, taus=None) -> np.ndarray:
        loss = np.zeros(self.local, dtype=np.float32)
        t, tp = self._taus(taus)
        _lib.check(_lib.lib().adpsgd_step(self._h, lr, tp, _ptr(loss, C.c_float)))
        return loss

    def step_host_batch(self, lr: float, feats: np.ndarray, labels: np.ndarray) -> np.ndarray:
        feats = np.ascontiguousarray(feats, dtype=np.float32)
        labels = np.ascontiguousarray(labels, dtype=np.int32)
        loss = np.zeros(self.local, dtype=np.float32)
        _lib.check(_lib.lib().adpsgd_step_host_batch(self._h, lr, _ptr(feats, C.c_float), _ptr(labels, C.c_int32),
                                                     _ptr(loss, C.c_float)))
        self._prefetched = [b for b in getattr(self, "_prefetched", []) if b[0] is not feats]
        return loss

    def prefetch_host_batch(self, feats: np.ndarray, labels: np.ndarray) -> None:
        """Queue the H2D copy of the next host batch so it overlaps the current step; pass the
        same (C-contiguous float32 / int32) arrays to the matching step_host_batch."""
        if not (feats.flags.c_contiguous and feats.dtype == np.float32 and labels.flags.c_contiguous
                and labels.dtype == np.int32):
            raise ValueError("prefetch_host_batch needs C-contiguous float32 features and int32 labels")
        _lib.check(_lib.lib().adpsgd_prefetch_host_batch(self._h, _ptr(feats, C.c_float), _ptr(labels, C.c_int32)))
        if not hasattr(self, "_prefetched"):
            self._prefetched = []
        self._prefetched.append((feats, labels))  # keep the host memory alive until its step

    def step_injected(self, lr: float, grads: np.ndarray, taus=None) -> None:
        g = np.ascontiguousarray(grads, dtype=np.float64)
        t, tp = self._taus(taus)
        _lib.check(_lib.lib().adpsgd_step_injected(self._h, lr, tp, _ptr(g, C.c_double)))

    def gradient(self, w, idx):
        w = np.ascontiguousarray(w, dtype=np.float64)
        idx = np.ascontiguousarray(idx, dtype=np.int32)
        g = np.zeros(self.D, dtype=np.float64)
        loss = C.c_double()
        _lib.check(_lib.lib().adpsgd_gradient(self._h, _ptr(w, C.c_double), _ptr(idx, C.c_int32), len(idx),
                                              _ptr(g, C.c_double), C.byref(loss)))
        return loss.value, g

    def set_straggler(self, j: int, factor: float) -> None:
        _lib.check(_lib.lib().adpsgd_set_straggler(self._h, j, factor))

    def stats(self) -> dict:
        p = _lib.Perf()
        _lib.check(_lib.lib().adpsgd_get_stats(self._h, C.byref(p)))
        return {"last_step_ms": p.last_step_ms, "last_mix_ms": p.last_mix_ms, "gossip_bytes": p.gossip_bytes,
                "steps": p.steps, "kernel_launches": p.kernel_launches, "comm_start_ms": p.comm_start_ms,
                "comm_end_ms": p.comm_end_ms, "compute_end_ms": p.compute_end_ms}

    def consensus_distance(self) -> float:
        out = C.c_double()
        _lib.check(_lib.lib().adpsgd_consensus_distance(self._h, C.byref(out)))
        return out.value

    def averaged_model(self) -> np.ndarray:
        out = np.zeros(self.D, dtype=np.float64)
        _lib.check(_lib.lib().adpsgd_averaged_model(self._h, _ptr(out, C.c_double), self.D))
        return out

    def averaged_model_all(self) -> np.ndarray:
        """averaged_model over every global learner (peers mapped over NVLink included)."""
        out = np.zeros(self.D, dtype=np.float64)
        _lib.check(_lib.lib().adpsgd_averaged_model_all(self._h, _ptr(out, C.c_double), self.D))
        return out

    def consensus_gram(self, begin: int, end: int) -> np.ndarray:
        """Shard [begin, end) of the Gram of all global learners' deviations from their mean."""
        L = self.cfg.learners
        out = np.zeros(L * L, dtype=np.float64)
        _lib.check(_lib.lib().adpsgd_consensus_gram(self._h, begin, end, _ptr(out, C.c_double)))
        return out.reshape(L, L)

    def eval_loss(self, w, idx) -> float:
        w = np.ascontiguousarray(w, dtype=np.float64)
        idx = np.ascontiguousarray(idx, dtype=np.int32)
        out = C.c_double()
        _lib.check(_lib.lib().adpsgd_eval_loss(self._h, _ptr(w, C.c_double), _ptr(idx, C.c_int32), len(idx),
                                               C.byref(out)))
        return out.value

    # ---- multi-process plumbing (one process per GPU) ----
    def comm_init(self, rank: int, world: int, nccl_id: bytes | None) -> None:
        """nccl_id None: CUDA-IPC-only transport (FM/RM; steps separated by a host barrier)."""
        buf = None if nccl_id is None else C.create_string_buffer(nccl_id, 128)
        _lib.check(_lib.lib().adpsgd_comm_init(self._h, rank, world, buf))

    def export_ipc(self) -> bytes:
        n = int(_lib.lib().adpsgd_ipc_handle_size(self._h))
        buf = C.create_string_buffer(n)
        _lib.check(_lib.lib().adpsgd_export_ipc(self._h, buf, n))
        return buf.raw

    def import_ipc(self, rank: int, first: int, count: int, handles: bytes) -> None:
        buf = C.create_string_buffer(handles, len(handles))
        _lib.check(_lib.lib().adpsgd_import_ipc(self._h, rank, first, count, buf, len(handles)))

    def set_gossip_mode(self, mode: int) -> None:
        _lib.check(_lib.lib().adpsgd_set_gossip_mode(self._h, mode))

    def barrier(self) -> None:
        _lib.check(_lib.lib().adpsgd_barrier(self._h))

    def async_init(self, mode: "AsyncMode" = None, max_lag: int = 0, timeout_s: float = 60.0) -> None:
        """Free-running async FM / RM (one learner per process): switch to the 4-slot publication
        ring (call before export_ipc)."""
        mode = AsyncMode.FREE if mode is None else AsyncMode(mode)
        _lib.check(_lib.lib().adpsgd_async_init(self._h, int(mode), max_lag, timeout_s))

    def async_step(self, lr: float):
        """One free-running iteration (no barrier): returns (loss, info dict: versions mixed with,
        neighbours, torn-read retries, wait / step device ms)."""
        loss = C.c_float()
        info = _lib.AsyncInfo()
        _lib.check(_lib.lib().adpsgd_async_step(self._h, lr, C.byref(loss), C.byref(info)))
        return float(loss.value), {f: getattr(info, f) for f, _ in _lib.AsyncInfo._fields_ if f != "reserved"}

    def last_gradient(self) -> np.ndarray:
        """fp32 gradient of local learner 0's last step (diagnosis / async-consistency tests)."""
        out = np.empty(self.D, dtype=np.float32)
        _lib.check(_lib.lib().adpsgd_debug_buffer(self._h, 103, out.ctypes.data_as(C.c_void_p), out.nbytes))
        return out

    def set_step_delay(self, j: int, ms: float, on_host: bool = False) -> None:
        _lib.check(_lib.lib().adpsgd_set_step_delay(self._h, j, ms, int(on_host)))

    def gossip_probe(self, left: int = -1, right: int = -1, reps: int = 5) -> dict:
        """Bandwidth of the FM/RM gossip path at this model size (adpsgd_gossip_probe): the fused
        mix kernel reading learners `left` / `right` (peers over NVLink, or local stand-ins at -1) and a
        copy-engine pull of both neighbours."""
        out = (C.c_double * 4)()
        _lib.check(_lib.lib().adpsgd_gossip_probe(self._h, left, right, reps, out))
        mix_ms, nvlink_bytes, copy_ms, mix_bytes = out[0], out[1], out[2], out[3]
        return {"mix_ms": mix_ms, "mix_hbm_gbs": mix_bytes / (mix_ms * 1e6) if mix_ms > 0 else None,
                "mix_nvlink_gbs": nvlink_bytes / (mix_ms * 1e6) if mix_ms > 0 and nvlink_bytes else None,
                "nvlink_bytes": nvlink_bytes, "copy_ms": copy_ms,
                "copy_gbs": 8.0 * self.D / (copy_ms * 1e6) if copy_ms > 0 else None}


class DeviceGroup:
    """engine::run_training's vector<LearnerState> spread over several GPUs of ONE process
    (engine.cpp:212-304): one context per entry of `devices`, hosting a contiguous share of the
    cfg.learners learners, linked so that each reads the others' models (and SDPSGD gradients) in
    place over NVLink (adpsgd_group_link); step() runs every GPU concurrently (adpsgd_group_step)."""

    def __init__(self, model: ModelDesc, cfg: StrategyConfig, devices, precision: Precision = Precision.BF16,
                 shares=None):
        cfg.validate()
        n = len(devices)
        if shares is None:
            q, r = divmod(cfg.learners, n)
            shares = [q + (1 if i < r else 0) for i in range(n)]
        if sum(shares) != cfg.learners or min(shares) < 1:
            raise ConfigError("device group: shares must be >= 1 and sum to cfg.learners")
        self.cfg, self.model = cfg, model
        self.groups, first = [], 0
        for dev, cnt in zip(devices, shares):
            self.groups.append(LearnerGroup(model, cfg, precision=precision, device=dev, first_learner=first,
                                            local_learners=cnt))
            first += cnt
        self._arr = (C.c_void_p * n)(*[g.handle for g in self.groups])
        _lib.check(_lib.lib().adpsgd_group_link(self._arr, n))
        self.D = self.groups[0].D

    def _owner(self, gid: int):
        for g in self.groups:
            if g.first <= gid < g.first + g.local:
                return g, gid - g.first
        raise InvalidStateError(f"learner {gid} outside the group")

    def set_dataset(self, feats, labels, train_count: int) -> None:
        for g in self.groups:
            g.set_dataset(feats, labels, train_count)

    def step(self, lr: float) -> np.ndarray:
        loss = np.zeros(self.cfg.learners, dtype=np.float32)
        _lib.check(_lib.lib().adpsgd_group_step(self._arr, len(self.groups), lr, _ptr(loss, C.c_float)))
        return loss

    def weights(self, gid: int) -> np.ndarray:
        g, j = self._owner(gid)
        return g.weights(j)

    def averaged_model(self) -> np.ndarray:
        return self.groups[0].averaged_model_all()

    def consensus_distance(self) -> float:
        """Each context reduces its share of the parameters over every learner (peer loads), the
        shards are summed on the host (mixing.cpp:159-180)."""
        from .dist import shard_range
        G = sum(g.consensus_gram(*shard_range(self.D, i, len(self.groups))) for i, g in enumerate(self.groups))
        return consensus_from_gram(G)

    def close(self) -> None:
        for g in self.groups:
            g.close()


def consensus_from_gram(gram) -> float:
    """sqrt(lambda_max) of a consensus Gram (mixing.cpp:174-179)."""
    G = np.ascontiguousarray(gram, dtype=np.float64)
    out = C.c_double()
    _lib.check(_lib.lib().adpsgd_consensus_from_gram(_ptr(G, C.c_double), G.shape[0], C.byref(out)))
    return float(out.value)


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    _lib.check(_lib.lib().adpsgd_nccl_unique_id(buf))
    return buf.raw


class LstmObjective:
    """objectives::Objective (objectives.hpp:45-69) for the BLSTM, evaluated on the GPU.
    loss/gradient take a flat fp64 parameter vector and a batch of segment indices."""

    def __init__(self, group: LearnerGroup):
        self.g = group

    def dimension(self) -> int:
        return self.g.D

    def gradient(self, w, indices) -> np.ndarray:
        return self.g.gradient(w, indices)[1]

    def loss(self, w, indices) -> float:
        return self.g.gradient(w, indices)[0]


# ---------------------------------------------------------------------------
# run_training (engine.cpp:206-304) and its record / CSV output (engine.hpp:107-125, csvio.hpp)
# ---------------------------------------------------------------------------
DIVERGENCE_FACTOR = 10.0  # engine.cpp:15


@dataclass
class RunRecord:
    iterations: list = field(default_factory=list)   # (k, consensus, lr)
    epochs: list = field(default_factory=list)       # (epoch, heldout_loss, train_loss, lr)
    final_model: np.ndarray | None = None
    diverged: bool = False
    divergence_epoch: int = -1
    iteration_count: int = 0


def iterations_per_epoch(cfg: StrategyConfig, train_count: int) -> int:
    per = train_count // (cfg.learners * cfg.batch)  # engine.cpp:206-210
    return per if per > 0 else 1


def run_training(cfg: StrategyConfig, model: ModelDesc, feats, labels, train_count: int,
                 precision: Precision = Precision.BF16, device: int = 0, consensus_every: int = 1,
                 eval_train: bool = True, synth: tuple | None = None) -> RunRecord:
    """engine::run_training on the device: every local learner on one GPU, the mixing of
    cfg.strategy each iteration, consensus distance (every `consensus_every` iterations; the
    reference measures every iteration), per-epoch heldout / full-train loss of the averaged
    model and the divergence rule (non-finite or > 10x the initial heldout loss).
    synth = (n_seg, seed): with feats None, the device-generated synthetic dataset instead."""
    cfg.validate()
    g = LearnerGroup(model, cfg, precision=precision, device=device)
    try:
        if feats is None:
            n_seg, seed = synth
            g.synth_dataset(n_seg, train_count, seed)
        else:
            g.set_dataset(feats, labels, train_count)
            n_seg = np.asarray(feats).shape[0]
        heldout_idx = np.arange(train_count, n_seg, dtype=np.int32)
        train_idx = np.arange(train_count, dtype=np.int32)
        rec = RunRecord()
        initial = g.eval_loss(g.averaged_model(), heldout_idx) if len(heldout_idx) else float("nan")
        ipe = iterations_per_epoch(cfg, train_count)
        taus = list(cfg.staleness) if cfg.staleness else None
        k = 0
        for epoch in range(cfg.epochs):
            lr = lr_at(cfg.lr, epoch)
            for _ in range(ipe):
                g.step(lr, taus=taus if cfg.strategy == Strategy.GENERIC else None)
                cons = 0.0
                if cfg.learners > 1 and (k % consensus_every == 0):
                    cons = g.consensus_distance()
                rec.iterations.append((k, cons, lr))
                k += 1
            avg = g.averaged_model()
            heldout = g.eval_loss(avg, heldout_idx) if len(heldout_idx) else float("nan")
            train = g.eval_loss(avg, train_idx) if eval_train else float("nan")
            rec.epochs.append((epoch, heldout, train, lr))
            if not np.isfinite(heldout) or heldout > DIVERGENCE_FACTOR * initial:
                rec.diverged = True
                rec.divergence_epoch = epoch
                break
        rec.iteration_count = len(rec.iterations)
        rec.final_model = g.averaged_model()
        return rec
    finally:
        g.close()


def fmt_double(x: float) -> str:
    """csvio.hpp:12-16 (%.17g)."""
    return "%.17g" % x


def write_csv(record: RunRecord, out_dir: str, stem: str = "") -> None:
    """<stem>run.csv (epoch,heldout_loss,lr) and <stem>consensus.csv (k,distance): the reference
    CLI's write_run_outputs (tools/main.cpp:99-105), floats at 17 significant digits."""
    import os
    os.makedirs(out_dir, exist_ok=True)
    with open(os.path.join(out_dir, stem + "run.csv"), "w") as f:
        f.write("epoch,heldout_loss,lr\n")
        for e, h, _t, lr in record.epochs:
            f.write(f"{e},{fmt_double(h)},{fmt_double(lr)}\n")
    with open(os.path.join(out_dir, stem + "consensus.csv"), "w") as f:
        f.write("k,distance\n")
        for k, c, _lr in record.iterations:
            f.write(f"{k},{fmt_double(c)}\n")
