"""Generate the committed golden fixtures in tests/golden/ (run HERE, in the build container).

* pairing.json — from oracle/_ref/libref_rng.so, i.e. the reference's OWN
  proj/include/adpsgd/rng.hpp compiled in place, wrapped by the 6-line Fisher-Yates
  restatement of proj/src/mixing.cpp:72-76 (Eigen is absent, so mixing.cpp itself
  cannot be compiled). Permutation sequences, seed derivations, w0 and learner
  batch streams.
* lstm_<name>.npz — fp64 loss and flat gradient of the BLSTM acoustic model computed
  by torch.nn.LSTM / nn.Linear / cross_entropy on CPU (the reference has no LSTM:
  SPEC.md:9), for small shapes, with the same flat parameter layout as the oracle.

Usage: python tests/golden/make_golden.py
"""
from __future__ import annotations

import ctypes as C
import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402

SEEDS = [0, 7, 1234, 2025]
ORDERS = list(range(3, 17)) + [64]
LONG_K = 10000


def _perm(R, seed, L, k):
    out = np.zeros(L, dtype=np.int32)
    R.ref_permutation_for_iteration(seed, L, k, out.ctypes.data_as(C.POINTER(C.c_int32)))
    return out


def pairing_fixture():
    R = O.ref_lib()
    if R is None:
        raise SystemExit("oracle/_ref/libref_rng.so missing: run `make -C oracle` with /root/reference mounted")
    fx = {"source": "reference proj/include/adpsgd/rng.hpp compiled in place (oracle/_ref)",
          "short": {}, "long_sha256": {}, "derive": {}, "w0": {}, "batches": {}}
    for s in SEEDS:
        for L in ORDERS + [1, 2]:
            fx["short"][f"{s}/{L}"] = [_perm(R, s, L, k).tolist() for k in range(16)]
    for s in SEEDS[:2]:
        for L in ORDERS:
            h = hashlib.sha256()
            for k in range(LONG_K):
                h.update(_perm(R, s, L, k).tobytes())
            fx["long_sha256"][f"{s}/{L}"] = h.hexdigest()
    fx["derive"] = {
        "derive_seed(0,0xC001)": str(R.ref_derive_seed(0, 0xC001)),
        "derive_seed(0,0xC001,0)": str(R.ref_derive_seed3(0, 0xC001, 0)),
        "derive_seed(1234,0xA001)": str(R.ref_derive_seed(1234, 0xA001)),
        "derive_seed(1234,0xB003)": str(R.ref_derive_seed(1234, 0xB000 + 3)),
        "mt19937_64(42)": str(R.ref_mt_first(42)),
    }
    w = np.zeros(16)
    R.ref_init_w0(1234, 16, w.ctypes.data_as(C.POINTER(C.c_double)))
    fx["w0"]["1234"] = [float.hex(float(x)) for x in w]
    for learner in range(4):
        b = np.zeros((5, 8), dtype=np.int32)
        R.ref_learner_batches(1234, learner, 5, 8, 1000, b.ctypes.data_as(C.POINTER(C.c_int32)))
        fx["batches"][f"1234/{learner}/M8/N1000"] = b.tolist()
    with open(os.path.join(HERE, "pairing.json"), "w") as f:
        json.dump(fx, f, indent=0, sort_keys=True)


LSTM_CASES = {
    # name: (layers, hidden, bidirectional, input_dim, proj, classes, unroll, M)
    "uni2": (2, 8, 0, 5, 0, 7, 5, 3),
    "bi2p": (2, 6, 1, 5, 4, 9, 4, 2),
    "bi3p_t21": (3, 16, 1, 12, 8, 11, 21, 2),
}


def torch_loss_grad(case, w, feats, labels, idx):
    import torch
    layers, H, bi, I, P, Cn, T, M = case
    d = O.desc(layers, H, bi, I, P, Cn, T)
    offs = O.param_offsets(d)
    nd = 2 if bi else 1
    lstm = torch.nn.LSTM(I, H, num_layers=layers, bidirectional=bool(bi), batch_first=True).double()
    top = H * nd
    proj = torch.nn.Linear(top, P).double() if P > 0 else None
    out = torch.nn.Linear(P if P > 0 else top, Cn).double()
    wt = torch.tensor(w)
    k = 0
    with torch.no_grad():
        for l in range(layers):
            in_l = I if l == 0 else top
            for dd in range(nd):
                sfx = f"l{l}" + ("_reverse" if dd == 1 else "")
                o_ih, o_hh, o_b = offs[k], offs[k + 1], offs[k + 2]
                k += 3
                getattr(lstm, f"weight_ih_{sfx}").copy_(wt[o_ih:o_ih + 4 * H * in_l].view(4 * H, in_l))
                getattr(lstm, f"weight_hh_{sfx}").copy_(wt[o_hh:o_hh + 4 * H * H].view(4 * H, H))
                getattr(lstm, f"bias_ih_{sfx}").copy_(wt[o_b:o_b + 4 * H])
                getattr(lstm, f"bias_hh_{sfx}").zero_()
        if P > 0:
            proj.weight.copy_(wt[offs[k]:offs[k] + P * top].view(P, top))
            proj.bias.copy_(wt[offs[k + 1]:offs[k + 1] + P])
            k += 2
        oin = P if P > 0 else top
        out.weight.copy_(wt[offs[k]:offs[k] + Cn * oin].view(Cn, oin))
        out.bias.copy_(wt[offs[k + 1]:offs[k + 1] + Cn])
    x = torch.tensor(feats[idx].astype(np.float64))          # [M, T, I]
    y = torch.tensor(labels[idx].astype(np.int64))           # [M, T]
    h, _ = lstm(x)
    if proj is not None:
        h = proj(h)
    logits = out(h)
    loss = torch.nn.functional.cross_entropy(logits.reshape(-1, Cn), y.reshape(-1))
    loss.backward()
    g = np.zeros_like(w)
    k = 0
    for l in range(layers):
        in_l = I if l == 0 else top
        for dd in range(nd):
            sfx = f"l{l}" + ("_reverse" if dd == 1 else "")
            o_ih, o_hh, o_b = offs[k], offs[k + 1], offs[k + 2]
            k += 3
            g[o_ih:o_ih + 4 * H * in_l] = getattr(lstm, f"weight_ih_{sfx}").grad.numpy().ravel()
            g[o_hh:o_hh + 4 * H * H] = getattr(lstm, f"weight_hh_{sfx}").grad.numpy().ravel()
            g[o_b:o_b + 4 * H] = getattr(lstm, f"bias_ih_{sfx}").grad.numpy().ravel()
    if P > 0:
        g[offs[k]:offs[k] + P * top] = proj.weight.grad.numpy().ravel()
        g[offs[k + 1]:offs[k + 1] + P] = proj.bias.grad.numpy().ravel()
        k += 2
    oin = P if P > 0 else top
    g[offs[k]:offs[k] + Cn * oin] = out.weight.grad.numpy().ravel()
    g[offs[k + 1]:offs[k + 1] + Cn] = out.bias.grad.numpy().ravel()
    return float(loss.item()), g


def lstm_fixtures():
    for name, case in LSTM_CASES.items():
        layers, H, bi, I, P, Cn, T, M = case
        d = O.desc(layers, H, bi, I, P, Cn, T)
        D = O.param_count(d)
        rng = np.random.default_rng(abs(hash(name)) % (2 ** 32) if False else sum(map(ord, name)))
        w = rng.normal(0.0, 0.3, size=D)
        n_seg = 6
        feats = rng.normal(0.0, 1.0, size=(n_seg, T, I)).astype(np.float32)
        labels = rng.integers(0, Cn, size=(n_seg, T)).astype(np.int32)
        idx = rng.integers(0, n_seg, size=M).astype(np.int32)
        loss, g = torch_loss_grad(case, w, feats, labels, idx)
        np.savez(os.path.join(HERE, f"lstm_{name}.npz"), case=np.array(case, dtype=np.int64), w=w,
                 feats=feats, labels=labels, idx=idx, loss=np.array(loss), grad=g)


if __name__ == "__main__":
    pairing_fixture()
    lstm_fixtures()
    print("golden fixtures written to", HERE)
