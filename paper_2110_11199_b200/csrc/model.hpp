// Flat parameter layout of the BLSTM acoustic model — identical to the oracle's
// (oracle/adpsgd_oracle.cpp make_layout) and to torch.nn.LSTM's per-tensor layout:
// per layer, per direction: W_ih[4H x I_l] (row-major), W_hh[4H x H], b[4H] (gate
// order i,f,g,o; one merged bias); then W_proj[P x nd*H], b_proj[P] (if P > 0); then
// W_out[C x (P or nd*H)], b_out[C].
#pragma once

#include <cstdint>
#include <vector>

#include "adpsgd_b200.h"

namespace ab {

struct DirOff { int64_t w_ih, w_hh, b; };

struct Layout {
    int L = 0, H = 0, nd = 1, I = 0, P = 0, C = 0, T = 0;
    std::vector<int> in_dim;               // per layer
    std::vector<std::vector<DirOff>> dir;  // [layer][dir]
    int64_t w_proj = -1, b_proj = -1, w_out = 0, b_out = 0, total = 0;
    int top = 0, out_in = 0;
};

inline Layout make_layout(const adpsgd_model_desc& m) {
    Layout Lo;
    Lo.L = m.layers; Lo.H = m.hidden; Lo.nd = m.bidirectional ? 2 : 1; Lo.I = m.input_dim;
    Lo.P = m.proj; Lo.C = m.classes; Lo.T = m.unroll;
    const int64_t H = m.hidden;
    int64_t off = 0;
    for (int l = 0; l < m.layers; ++l) {
        const int in = l == 0 ? m.input_dim : static_cast<int>(H * Lo.nd);
        Lo.in_dim.push_back(in);
        std::vector<DirOff> ds;
        for (int d = 0; d < Lo.nd; ++d) {
            DirOff o;
            o.w_ih = off; off += 4 * H * in;
            o.w_hh = off; off += 4 * H * H;
            o.b = off; off += 4 * H;
            ds.push_back(o);
        }
        Lo.dir.push_back(ds);
    }
    Lo.top = static_cast<int>(H * Lo.nd);
    if (m.proj > 0) {
        Lo.w_proj = off; off += static_cast<int64_t>(m.proj) * Lo.top;
        Lo.b_proj = off; off += m.proj;
        Lo.out_in = m.proj;
    } else {
        Lo.out_in = Lo.top;
    }
    Lo.w_out = off; off += static_cast<int64_t>(m.classes) * Lo.out_in;
    Lo.b_out = off; off += m.classes;
    Lo.total = off;
    return Lo;
}

// Forward FLOPs per frame (GEMMs only) and training FLOPs per frame
// (3 x forward minus the layer-1 input dgrad, which is never computed).
inline double fwd_flops_per_frame(const Layout& Lo) {
    double f = 0;
    for (int l = 0; l < Lo.L; ++l) f += 2.0 * Lo.nd * 4.0 * Lo.H * (Lo.in_dim[l] + Lo.H);
    if (Lo.P > 0) f += 2.0 * Lo.top * Lo.P;
    f += 2.0 * Lo.out_in * Lo.C;
    return f;
}
inline double train_flops_per_frame(const Layout& Lo) {
    return 3.0 * fwd_flops_per_frame(Lo) - 2.0 * Lo.nd * 4.0 * Lo.H * Lo.in_dim[0];
}

}  // namespace ab
