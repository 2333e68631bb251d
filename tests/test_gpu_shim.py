"""GPU: the INTEGRATION.md shim as compiled C++ (tools/shim: b200::LstmObjective behind the
reference's own objectives::Objective interface, built against proj/include where it lies) --
loss / gradient / heldout_loss through the reference's virtual calls equal the library's, and a
library status surfaces as the reference's exception type (errors.hpp). The binary is built in
the build container (__graft_entry__.build) and travels with the repository snapshot."""
import os
import subprocess

import numpy as np
import pytest

from paper_2110_11199_b200 import LearnerGroup, ModelDesc, Precision, StrategyConfig

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tools", "shim", "build", "shim_demo")


@pytest.mark.skipif(not os.path.exists(BIN), reason="shim not built (reference headers absent at build time)")
@pytest.mark.parametrize("prec", [Precision.FP32, Precision.BF16])
def test_shim_objective_matches_library(tmp_path, prec):
    m = ModelDesc(layers=2, hidden=32, bidirectional=True, input_dim=20, proj=16, classes=24, unroll=6)
    rng = np.random.default_rng(11)
    n_seg, train, M = 40, 36, 4
    feats = rng.normal(size=(n_seg, m.unroll, m.input_dim)).astype(np.float32)
    labels = rng.integers(0, m.classes, size=(n_seg, m.unroll)).astype(np.int32)
    g = LearnerGroup(m, StrategyConfig(learners=1, batch=M, seed=2), precision=prec)
    g.set_dataset(feats, labels, train)
    w = g.weights(0)
    idx = np.array([3, 17, 0, 35], dtype=np.int32)
    hdr = np.array([m.layers, m.hidden, int(m.bidirectional), m.input_dim, m.proj, m.classes, m.unroll, int(prec), M,
                    n_seg, train, M], dtype=np.int32)
    inp, out = tmp_path / "in.bin", tmp_path / "out.bin"
    inp.write_bytes(hdr.tobytes() + feats.tobytes() + labels.tobytes() + w.astype(np.float64).tobytes() + idx.tobytes())
    r = subprocess.run([BIN, str(inp), str(out)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    res = np.frombuffer(out.read_bytes(), dtype=np.float64)
    loss, heldout, mapped, grad = res[0], res[1], res[2], res[3:]
    assert mapped == 1.0
    want_loss, want_g = g.gradient(w, idx)
    assert abs(loss - want_loss) <= 1e-6 * abs(want_loss)
    assert np.max(np.abs(grad - want_g)) <= 1e-6 * np.max(np.abs(want_g))
    want_h = g.eval_loss(w, np.arange(train, n_seg, dtype=np.int32))
    assert abs(heldout - want_h) <= 1e-6 * abs(want_h)
    g.close()
