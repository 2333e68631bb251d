"""Multi-process host logic of the one-process-per-GPU path, on CPU with gloo (world_size 2
and 4): rank->learner mapping, per-iteration neighbour plans agreed bit-exactly by every rank,
per-learner sampling streams, the handle all-gather protocol and max-over-ranks timing."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2110_11199_b200 import Strategy
from paper_2110_11199_b200 import dist as D


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update({"RANK": str(rank), "WORLD_SIZE": str(world), "LOCAL_RANK": str(rank),
                       "MASTER_ADDR": "127.0.0.1", "MASTER_PORT": str(port)})
    try:
        import sys
        sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
        from oracle import oracle as O
        env = D.rank_env()
        P = D.Plumbing(env)
        out = {"learner": env.learner}
        # every rank derives the RM plans itself; they must agree bit-exactly
        L = max(3, world)
        plans = [D.neighbour_plan(Strategy.ADPSGD_RM, 2025, L, k) for k in range(50)]
        for pl in plans:
            D.validate_plan(pl)
        gathered = P.all_gather_bytes(repr(plans).encode())
        out["plans_agree"] = all(g == gathered[0] for g in gathered)
        # the learner's sampling stream is the reference's stream 0xB000 + learner id
        ref = O.learner_batches(7, env.learner, 3, 16, 1000)
        blob = P.all_gather_bytes(ref.tobytes())
        out["streams_distinct"] = len(set(blob)) == world
        out["stream_matches_oracle"] = np.frombuffer(blob[env.rank], dtype=np.int32).reshape(3, 16).tolist() == ref.tolist()
        # id broadcast + handle exchange protocol (opaque bytes, ordered by rank)
        nid = P.broadcast_bytes(b"nccl-id-" + bytes([env.rank]) if env.rank == 0 else None)
        out["id_from_rank0"] = nid == b"nccl-id-\x00"
        hs = P.all_gather_bytes(bytes([env.rank]) * 128)
        out["handles_in_rank_order"] = [h[0] for h in hs] == list(range(world))
        out["max"] = P.max_over_ranks(float(env.rank) * 1.5)
        P.barrier()
        q.put((rank, out))
    except Exception as e:  # pragma: no cover - surfaced by the parent
        q.put((rank, {"error": repr(e)}))


@pytest.mark.parametrize("world", [2, 4])
def test_gloo_plumbing(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=240) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    for r in range(world):
        o = res[r]
        assert "error" not in o, o
        assert o["learner"] == r
        assert o["plans_agree"] and o["streams_distinct"] and o["stream_matches_oracle"]
        assert o["id_from_rank0"] and o["handles_in_rank_order"]
        assert o["max"] == 1.5 * (world - 1)


def test_rank_env_and_plans():
    e = D.rank_env({"WORLD_SIZE": "8", "RANK": "5", "LOCAL_RANK": "5"})
    assert (e.rank, e.world, e.local_rank, e.learner) == (5, 8, 5, 5)
    with pytest.raises(ValueError):
        D.rank_env({"WORLD_SIZE": "2", "RANK": "2"})
    fm = D.neighbour_plan(Strategy.ADPSGD_FM, 0, 8, 3)
    assert fm[0] == (7, 1) and fm[7] == (6, 0)
    for k in range(200):
        D.validate_plan(D.neighbour_plan(Strategy.ADPSGD_RM, 11, 8, k))
    with pytest.raises(ValueError):
        D.validate_plan([(1, 2), (0, 2), (1, 0)][:2] + [(0, 0)])
    with pytest.raises(ValueError):
        D.neighbour_plan(Strategy.ADPSGD_D1D, 0, 8, 0)


def test_gossip_bytes():
    D_ = 145145344
    assert D.gossip_ingress_bytes(Strategy.ADPSGD_FM, D_, 8) == 8 * D_
    assert D.gossip_ingress_bytes(Strategy.ADPSGD_D1D, D_, 8) == int(2 * 7 / 8 * 4 * D_)
    assert D.gossip_ingress_bytes(Strategy.ADPSGD_RM, D_, 1) == 0


def test_shard_ranges_cover_parameters():
    for D_, world in ((145145344, 8), (10, 3), (2, 4), (0, 2)):
        rs = [D.shard_range(D_, r, world) for r in range(world)]
        assert rs[0][0] == 0 and rs[-1][1] == D_
        assert all(a[1] == b[0] for a, b in zip(rs, rs[1:]))
        assert max(e - b for b, e in rs) - min(e - b for b, e in rs) <= 1


def _gram_worker(rank, world, port, q):
    os.environ.update({"RANK": str(rank), "WORLD_SIZE": str(world), "LOCAL_RANK": str(rank),
                       "MASTER_ADDR": "127.0.0.1", "MASTER_PORT": str(port)})
    try:
        P = D.Plumbing(D.rank_env())
        rng = np.random.default_rng(0)
        W = rng.normal(size=(3, 101))  # 3 learners' models, the same on every rank
        b, e = D.shard_range(101, rank, world)
        dev = W[:, b:e] - W[:, b:e].mean(axis=0)
        G = D.reduce_gram(dev @ dev.T, P)
        P.barrier()
        q.put((rank, G))
    except Exception as e:  # pragma: no cover
        q.put((rank, repr(e)))


@pytest.mark.parametrize("world", [2, 4])
def test_sharded_gram_sums_to_full_gram(world):
    """The multi-rank consensus distance: per-rank Gram shards summed by the gloo allreduce equal
    the Gram over the whole parameter vector (mixing.cpp:159-180)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_gram_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in ps:
        p.join(timeout=60)
    W = np.random.default_rng(0).normal(size=(3, 101))
    dev = W - W.mean(axis=0)
    for r in range(world):
        assert not isinstance(res[r], str), res[r]
        assert np.allclose(res[r], dev @ dev.T, rtol=1e-12, atol=1e-12)
