"""One-process-per-GPU plumbing for the learner step (host side only).

Each rank hosts exactly one learner (global id = rank) on GPU LOCAL_RANK. torch.distributed
(gloo) is plumbing: it broadcasts the NCCL unique id and all-gathers the CUDA-IPC handles of
every learner's double-buffered weights; the data path (NVLink peer loads for FM/RM, NCCL
allreduce for D1D / SDPSGD) lives in the C++ library. Timing is reduced as the max over ranks.

The pure functions here (env parsing, the per-iteration neighbour plan, plan validation,
handle bookkeeping) are what tests/test_dist.py exercises with gloo at world_size 2 and 4.
"""
from __future__ import annotations

import os
from dataclasses import dataclass

from .engine import Strategy, pairing


@dataclass(frozen=True)
class RankEnv:
    rank: int
    world: int
    local_rank: int

    @property
    def learner(self) -> int:
        return self.rank


def rank_env(environ=None) -> RankEnv:
    e = os.environ if environ is None else environ
    world = int(e.get("WORLD_SIZE", "1"))
    rank = int(e.get("RANK", "0"))
    local = int(e.get("LOCAL_RANK", str(rank)))
    if not (0 <= rank < world):
        raise ValueError(f"RANK {rank} outside WORLD_SIZE {world}")
    return RankEnv(rank, world, local)


def neighbour_plan(strategy: Strategy, seed: int, learners: int, k: int):
    """(left, right) of every learner at iteration k — the pairs whose weights each GPU pulls
    over NVLink. FM: l±1 (mixing.cpp:35-50); RM: the Fisher-Yates ring of iteration k
    (engine.cpp:130-134, chronos.cpp:227-235)."""
    if strategy not in (Strategy.ADPSGD_FM, Strategy.ADPSGD_RM):
        raise ValueError("neighbour plans exist for FM / RM only")
    return pairing(strategy, seed, learners, k)[1]


def validate_plan(plan) -> None:
    """A ring plan is symmetric (j is i's left iff i is j's right), has no self-loops and
    every learner appears exactly once as someone's left and once as someone's right."""
    L = len(plan)
    lefts = sorted(p[0] for p in plan)
    rights = sorted(p[1] for p in plan)
    if lefts != list(range(L)) or rights != list(range(L)):
        raise ValueError("ring plan is not a permutation")
    for i, (l, r) in enumerate(plan):
        if l == i or r == i:
            raise ValueError(f"learner {i} paired with itself")
        if plan[l][1] != i or plan[r][0] != i:
            raise ValueError(f"asymmetric pairing at learner {i}")


def gossip_ingress_bytes(strategy: Strategy, params: int, learners: int) -> int:
    """Bytes a GPU pulls per iteration: FM/RM 2 neighbours x fp32 model; D1D/SDPSGD the
    ring-allreduce bus bytes 2 (L-1)/L x 4 D."""
    if learners == 1:
        return 0
    if strategy in (Strategy.ADPSGD_FM, Strategy.ADPSGD_RM):
        return 2 * 4 * params
    return int(2 * (learners - 1) / learners * 4 * params)


class Plumbing:
    """torch.distributed-backed exchange of the NCCL id and IPC handles (gloo for plumbing)."""

    def __init__(self, env: RankEnv):
        import torch.distributed as dist
        self.env = env
        self.dist = dist
        if env.world > 1 and not dist.is_initialized():
            dist.init_process_group("gloo")

    def broadcast_bytes(self, blob: bytes | None) -> bytes:
        if self.env.world == 1:
            return blob
        obj = [blob if self.env.rank == 0 else None]
        self.dist.broadcast_object_list(obj, src=0)
        return obj[0]

    def all_gather_bytes(self, blob: bytes) -> list:
        if self.env.world == 1:
            return [blob]
        out = [None] * self.env.world
        self.dist.all_gather_object(out, blob)
        return out

    def max_over_ranks(self, value: float) -> float:
        if self.env.world == 1:
            return value
        import torch
        t = torch.tensor([value], dtype=torch.float64)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t[0])

    def barrier(self) -> None:
        if self.env.world > 1:
            self.dist.barrier()


def connect(group, plumbing: Plumbing) -> None:
    """Wire a LearnerGroup (one learner per rank) into the multi-GPU ring: NCCL communicator
    from rank 0's id, then every peer's weight buffers mapped through CUDA IPC."""
    from .engine import nccl_unique_id
    env = plumbing.env
    if env.world == 1:
        return
    nid = plumbing.broadcast_bytes(nccl_unique_id() if env.rank == 0 else None)
    group.comm_init(env.rank, env.world, nid)
    handles = plumbing.all_gather_bytes(group.export_ipc())
    for r, h in enumerate(handles):
        group.import_ipc(r, r, 1, h)


def shard_range(D: int, rank: int, world: int):
    """Contiguous parameter shard [begin, end) of rank (sizes differ by at most one)."""
    if not (0 <= rank < world):
        raise ValueError("rank outside world")
    q, r = divmod(D, world)
    begin = rank * q + min(rank, r)
    return begin, begin + q + (1 if rank < r else 0)


def reduce_gram(partial, plumbing: "Plumbing"):
    """Sum the ranks' consensus-Gram shards (a small gloo allreduce on the host)."""
    import numpy as np
    G = np.ascontiguousarray(partial, dtype=np.float64)
    if plumbing.env.world == 1:
        return G
    import torch
    t = torch.from_numpy(G.copy())
    plumbing.dist.all_reduce(t)
    return t.numpy()


def consensus_distance(group, plumbing: "Plumbing") -> float:
    """mixing.cpp:159-180 across ranks (one learner per GPU, engine.cpp:284-289): each rank reads
    1/world of every learner's model -- its own from HBM, the others over NVLink -- into a Gram
    shard; the shards are summed across ranks and the largest eigenvalue taken."""
    from .engine import consensus_from_gram
    b, e = shard_range(group.D, plumbing.env.rank, plumbing.env.world)
    return consensus_from_gram(reduce_gram(group.consensus_gram(b, e), plumbing))
