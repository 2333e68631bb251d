"""Run configuration front-end: the reference's INI format (proj/src/config.cpp:99-277,
include/adpsgd/config.hpp) with the BLSTM objective added.

Sections [run], [engine], [lr], [objective], [cluster], [stragglers]; '#' starts a comment;
unknown sections or keys, malformed numbers and bad enum values raise ConfigError with the
reference's messages. resolved_text() writes every field with its default materialised, in the
reference's order and number format (%.17g), so a run can be repeated from its output directory.

Objective kinds: the reference's quadratic / logistic / mlp toy objectives parse (their keys are
kept and resolved) but are not built here -- the hot path of this build is the BLSTM acoustic
model, objective.kind = blstm, which adds the keys layers, bidirectional, proj, unroll and
precision (fp32 | bf16) next to the shared input_dim / hidden / classes / samples; the held-out
split is the reference's 10 % (objectives.cpp:18-23).
"""
from __future__ import annotations

import math
import re
from dataclasses import dataclass, field

from .chronos import ClusterProfile
from .engine import LrSchedule, MixKind, ModelDesc, Precision, Strategy, StrategyConfig, fmt_double, strategy_from_name, \
    strategy_name
from .errors import ConfigError

_SECTIONS = ("run", "engine", "lr", "objective", "cluster", "stragglers")
_INT = re.compile(r"[+-]?[0-9]+")
# what std::stod consumes in full: decimal (with exponent), hex floats, inf / infinity / nan[(chars)]
_DOUBLE = re.compile(r"[+-]?(?:(?:[0-9]+\.?[0-9]*|\.[0-9]+)(?:[eE][+-]?[0-9]+)?"
                     r"|0[xX](?:[0-9a-fA-F]+\.?[0-9a-fA-F]*|\.[0-9a-fA-F]+)(?:[pP][+-]?[0-9]+)?"
                     r"|(?i:inf(?:inity)?|nan(?:\([0-9A-Za-z_]*\))?))")
_MIX_NAMES = {"uniform": MixKind.UNIFORM, "fixed_ring": MixKind.FIXED_RING, "random_ring": MixKind.RANDOM_RING}
_OBJECTIVES = ("quadratic", "logistic", "mlp", "blstm")


def _trim(s: str) -> str:
    return s.strip(" \t\r")


def _split_csv(s: str) -> list:
    return [t for t in (_trim(x) for x in s.split(",")) if t]


def _parse_double(key: str, value: str) -> float:
    if not _DOUBLE.fullmatch(value):
        raise ConfigError(f"key '{key}': expected a number, got '{value}'")
    if value.lstrip("+-")[:2].lower() == "0x":
        v = float.fromhex(value)
    else:
        v = float(value.split("(")[0])
    if math.isinf(v) and not re.search(r"(?i)inf", value):  # std::stod throws out_of_range
        raise ConfigError(f"key '{key}': expected a number, got '{value}'")
    return v


def _parse_int(key: str, value: str) -> int:
    if not _INT.fullmatch(value) or not -(1 << 63) <= int(value) < (1 << 63):  # std::stol, 64-bit long
        raise ConfigError(f"key '{key}': expected an integer, got '{value}'")
    return int(value)


def _as_int32(v: int) -> int:  # static_cast<int>(long)
    return ((v + (1 << 31)) % (1 << 32)) - (1 << 31)


def _parse_bool(key: str, value: str) -> bool:
    if value in ("true", "1"):
        return True
    if value in ("false", "0"):
        return False
    raise ConfigError(f"key '{key}': expected true/false, got '{value}'")


def split_train_count(total: int, heldout_fraction: float = 0.1) -> int:
    """objectives.cpp:18-23 (std::lround: halves away from zero)."""
    x = total * heldout_fraction
    heldout = int(math.floor(x + 0.5)) if x >= 0 else -int(math.floor(-x + 0.5))
    heldout = max(heldout, 1)
    if heldout >= total:
        heldout = total - 1
    return total - heldout


@dataclass
class ObjectiveSpec:
    kind: str = "quadratic"
    dimension: int = 10
    condition_number: float = 10.0
    noise_sigma: float = 0.05
    samples: int = 2048
    input_dim: int = 5
    hidden: int = 16
    classes: int = 3
    # blstm
    layers: int = 2
    bidirectional: bool = True
    proj: int = 0
    unroll: int = 21
    precision: str = "bf16"

    def model(self) -> ModelDesc:
        if self.kind != "blstm":
            raise ConfigError(f"objective.kind = {self.kind}: the toy objectives are not part of this build "
                              "(objective.kind = blstm)")
        return ModelDesc(self.layers, self.hidden, self.bidirectional, self.input_dim, self.proj, self.classes,
                         self.unroll)

    def precision_enum(self) -> Precision:
        return Precision.BF16 if self.precision == "bf16" else Precision.FP32

    def train_count(self) -> int:
        return split_train_count(self.samples)


@dataclass
class RunConfig:
    kind: str = "train"
    seed: int = 0
    strategy: StrategyConfig = field(default_factory=StrategyConfig)
    objective: ObjectiveSpec = field(default_factory=ObjectiveSpec)
    cluster: ClusterProfile = field(default_factory=ClusterProfile)
    straggler_learner: int = -1
    straggler_factor: float = 1.0
    coupled: bool = False
    iterations_per_learner: int = 20
    straggler_factors: list = field(default_factory=lambda: [5.0, 10.0, 100.0])
    straggler_strategies: list = field(
        default_factory=lambda: [Strategy.ADPSGD_FM, Strategy.ADPSGD_RM, Strategy.ADPSGD_D1D])

    @staticmethod
    def parse_file(path: str) -> "RunConfig":
        try:
            with open(path) as f:
                text = f.read()
        except OSError:
            raise ConfigError("cannot open config file: " + path) from None
        return RunConfig.parse_text(text)

    @staticmethod
    def parse_text(text: str) -> "RunConfig":
        c = RunConfig()
        st, lr, ob, cl = c.strategy, c.strategy.lr, c.objective, c.cluster
        section = ""
        # std::getline: '\n' separates lines; a trailing newline does not start another one
        lines = text.split("\n")
        if lines and lines[-1] == "":
            lines.pop()
        for line_no, raw in enumerate(lines, 1):
            line = _trim(raw.split("#", 1)[0])
            if not line:
                continue
            if line[0] == "[":
                if line[-1] != "]":
                    raise ConfigError(f"line {line_no}: bad section header")
                section = _trim(line[1:-1])
                if section not in _SECTIONS:
                    raise ConfigError(f"unknown section [{section}]")
                continue
            if "=" not in line:
                raise ConfigError(f"line {line_no}: expected key = value")
            key, value = (_trim(x) for x in line.split("=", 1))
            q = section + "." + key
            i = lambda: _as_int32(_parse_int(q, value))  # noqa: E731
            d = lambda: _parse_double(q, value)  # noqa: E731
            if q == "run.kind":
                if value not in ("train", "stragglers"):
                    raise ConfigError("run.kind must be train or stragglers, got " + value)
                c.kind = value
            elif q == "run.seed":
                c.seed = _parse_int(q, value) % (1 << 64)
            elif q == "engine.strategy":
                st.strategy = strategy_from_name(value)
            elif q == "engine.learners":
                st.learners = i()
            elif q == "engine.batch":
                st.batch = i()
            elif q == "engine.epochs":
                st.epochs = i()
            elif q == "engine.staleness_cap":
                st.staleness_cap = i()
            elif q == "engine.staleness":
                st.staleness = [_as_int32(_parse_int(q, t)) for t in _split_csv(value)]
            elif q == "engine.generic_mix":
                if value not in _MIX_NAMES:
                    raise ConfigError("unknown mix kind: " + value)
                st.generic_mix = _MIX_NAMES[value]
            elif q == "lr.base_lr":
                lr.base_lr = d()
            elif q == "lr.peak_lr":
                lr.peak_lr = d()
            elif q == "lr.warmup_epochs":
                lr.warmup_epochs = i()
            elif q == "lr.anneal_factor":
                lr.anneal_factor = d()
            elif q == "lr.anneal_start_epoch":
                lr.anneal_start_epoch = i()
            elif q == "objective.kind":
                if value not in _OBJECTIVES:
                    raise ConfigError("objective.kind must be quadratic, logistic, mlp or blstm")
                ob.kind = value
            elif q == "objective.dimension":
                ob.dimension = i()
            elif q == "objective.condition_number":
                ob.condition_number = d()
            elif q == "objective.noise_sigma":
                ob.noise_sigma = d()
            elif q == "objective.samples":
                ob.samples = i()
            elif q == "objective.input_dim":
                ob.input_dim = i()
            elif q == "objective.hidden":
                ob.hidden = i()
            elif q == "objective.classes":
                ob.classes = i()
            elif q == "objective.layers":
                ob.layers = i()
            elif q == "objective.bidirectional":
                ob.bidirectional = _parse_bool(q, value)
            elif q == "objective.proj":
                ob.proj = i()
            elif q == "objective.unroll":
                ob.unroll = i()
            elif q == "objective.precision":
                if value not in ("fp32", "bf16"):
                    raise ConfigError("objective.precision must be fp32 or bf16, got " + value)
                ob.precision = value
            elif q == "cluster.compute_time":
                cl.compute_time = d()
            elif q == "cluster.comm_pairwise":
                cl.comm_pairwise = d()
            elif q == "cluster.comm_allreduce":
                cl.comm_allreduce = d()
            elif q == "cluster.sync_overhead":
                cl.sync_overhead = d()
            elif q == "cluster.coupled":
                c.coupled = _parse_bool(q, value)
            elif q == "cluster.iterations_per_learner":
                c.iterations_per_learner = i()
            elif q == "stragglers.factors":
                c.straggler_factors = [_parse_double(q, t) for t in _split_csv(value)]
            elif q == "stragglers.strategies":
                c.straggler_strategies = [strategy_from_name(t) for t in _split_csv(value)]
            elif q == "cluster.straggler_learner":
                c.straggler_learner = i()
            elif q == "cluster.straggler_factor":
                c.straggler_factor = d()
            else:
                raise ConfigError(f"unknown key '{key}' in section [{section}]")
        st.seed = c.seed
        cl.learners = st.learners
        if c.straggler_learner >= 0:
            cl.stragglers = [(c.straggler_learner, c.straggler_factor)]
        return c

    def resolved_text(self) -> str:
        """config.cpp:213-277, plus the blstm keys at the end of [objective]."""
        st, lr, ob, cl = self.strategy, self.strategy.lr, self.objective, self.cluster
        mix = {v: k for k, v in _MIX_NAMES.items()}[MixKind(st.generic_mix)]
        out = ["[run]", f"kind = {self.kind}", f"seed = {self.seed}", "", "[engine]",
               f"strategy = {strategy_name(st.strategy)}", f"learners = {st.learners}", f"batch = {st.batch}",
               f"epochs = {st.epochs}", f"staleness_cap = {st.staleness_cap}"]
        if st.staleness:
            out.append("staleness = " + ",".join(str(t) for t in st.staleness))
        out += [f"generic_mix = {mix}", "", "[lr]", f"base_lr = {fmt_double(lr.base_lr)}",
                f"peak_lr = {fmt_double(lr.peak_lr)}", f"warmup_epochs = {lr.warmup_epochs}",
                f"anneal_factor = {fmt_double(lr.anneal_factor)}", f"anneal_start_epoch = {lr.anneal_start_epoch}",
                "", "[objective]", f"kind = {ob.kind}", f"dimension = {ob.dimension}",
                f"condition_number = {fmt_double(ob.condition_number)}", f"noise_sigma = {fmt_double(ob.noise_sigma)}",
                f"samples = {ob.samples}", f"input_dim = {ob.input_dim}", f"hidden = {ob.hidden}",
                f"classes = {ob.classes}"]
        if ob.kind == "blstm":
            out += [f"layers = {ob.layers}", f"bidirectional = {'true' if ob.bidirectional else 'false'}",
                    f"proj = {ob.proj}", f"unroll = {ob.unroll}", f"precision = {ob.precision}"]
        out += ["", "[cluster]", f"compute_time = {fmt_double(cl.compute_time)}",
                f"comm_pairwise = {fmt_double(cl.comm_pairwise)}", f"comm_allreduce = {fmt_double(cl.comm_allreduce)}",
                f"sync_overhead = {fmt_double(cl.sync_overhead)}", f"straggler_learner = {self.straggler_learner}",
                f"straggler_factor = {fmt_double(self.straggler_factor)}",
                f"coupled = {'true' if self.coupled else 'false'}",
                f"iterations_per_learner = {self.iterations_per_learner}", "", "[stragglers]",
                "factors = " + ",".join(fmt_double(f) for f in self.straggler_factors),
                "strategies = " + ",".join(strategy_name(s) for s in self.straggler_strategies)]
        return "\n".join(out) + "\n"
