// Drives tools/shim/b200_shim.hpp through the reference's Objective interface: reads a problem
// written by tests/test_gpu_shim.py, evaluates loss / gradient / heldout_loss of the BLSTM on the
// device via the virtual calls a reference engine makes (engine.cpp:17-21, 291-299), writes the
// results back, and checks that a library error surfaces as the reference's exception type.
//   shim_demo <in.bin> <out.bin>
#include <cstdio>
#include <cstdint>
#include <fstream>
#include <iostream>
#include <memory>
#include <vector>

#include "b200_shim.hpp"

int main(int argc, char** argv) {
    if (argc != 3) {
        std::cerr << "usage: shim_demo <in.bin> <out.bin>\n";
        return 2;
    }
    std::ifstream in(argv[1], std::ios::binary);
    int32_t h[12];
    in.read(reinterpret_cast<char*>(h), sizeof(h));
    adpsgd_model_desc m{h[0], h[1], h[2], h[3], h[4], h[5], h[6]};
    const int precision = h[7], batch = h[8], n_seg = h[9], train_count = h[10], M = h[11];
    const int64_t D = adpsgd_param_count(&m);
    std::vector<float> feats(static_cast<size_t>(n_seg) * m.unroll * m.input_dim);
    std::vector<int32_t> labels(static_cast<size_t>(n_seg) * m.unroll);
    adpsgd::objectives::Vec w(D);
    adpsgd::objectives::SampleBatch batch_idx;
    batch_idx.indices.resize(M);
    in.read(reinterpret_cast<char*>(feats.data()), feats.size() * sizeof(float));
    in.read(reinterpret_cast<char*>(labels.data()), labels.size() * sizeof(int32_t));
    in.read(reinterpret_cast<char*>(w.data()), D * sizeof(double));
    in.read(reinterpret_cast<char*>(batch_idx.indices.data()), M * sizeof(int32_t));
    if (!in) {
        std::cerr << "short input\n";
        return 2;
    }
    // held as the reference holds it: Problem::objective is a shared_ptr<const Objective>
    std::shared_ptr<const adpsgd::objectives::Objective> obj =
        std::make_shared<b200::LstmObjective>(m, precision, batch, feats, labels, n_seg, train_count);
    if (obj->dimension() != D) {
        std::cerr << "dimension mismatch\n";
        return 1;
    }
    const adpsgd::objectives::Vec g = obj->gradient(w, batch_idx);
    const double loss = obj->loss(w, batch_idx);
    const double heldout = obj->heldout_loss(w);
    // a batch the context was not built for: DimensionError, as engine.cpp would see it
    bool mapped = false;
    try {
        adpsgd::objectives::SampleBatch wrong;
        wrong.indices.assign(batch_idx.indices.begin(), batch_idx.indices.end() - 1);
        (void)obj->gradient(w, wrong);
    } catch (const adpsgd::DimensionError&) {
        mapped = true;
    }
    std::ofstream out(argv[2], std::ios::binary);
    const double hdr[3] = {loss, heldout, mapped ? 1.0 : 0.0};
    out.write(reinterpret_cast<const char*>(hdr), sizeof(hdr));
    out.write(reinterpret_cast<const char*>(g.data()), D * sizeof(double));
    std::cout << "shim ok: D " << D << " loss " << loss << " heldout " << heldout
              << (mapped ? " DimensionError mapped" : " DimensionError NOT mapped") << "\n";
    return mapped ? 0 : 1;
}
