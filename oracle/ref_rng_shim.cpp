// TEST INFRASTRUCTURE ONLY — builds oracle/_ref/libref_rng.so from the reference's
// OWN header /root/reference/proj/include/adpsgd/rng.hpp (compiled where it lies,
// never copied). The rest of the reference (mixing.cpp, engine.cpp) needs Eigen 3,
// which is absent from this image (proj/CMakeLists.txt:22), so the 6-line Fisher-Yates
// loop of proj/src/mixing.cpp:72-76 and the stream tag of proj/src/engine.cpp:132 are
// restated here around the reference Rng. Used only to pin oracle/ and the product's
// pairing generator bit-exactly (tests/test_oracle.py, tests/golden/make_golden.py).
#include <cstdint>
#include <utility>
#include <vector>

#include "adpsgd/rng.hpp"

extern "C" {

uint64_t ref_derive_seed(uint64_t s, uint64_t a) { return adpsgd::derive_seed(s, a); }
uint64_t ref_derive_seed3(uint64_t s, uint64_t a, uint64_t b) { return adpsgd::derive_seed(s, a, b); }
uint64_t ref_mt_first(uint64_t seed) { adpsgd::Rng r(seed); return r.next_u64(); }

void ref_permutation_for_iteration(uint64_t seed, int L, int64_t k, int32_t* mapping) {
    adpsgd::Rng rng(adpsgd::derive_seed(seed, 0xC001, static_cast<uint64_t>(k)));
    for (int i = 0; i < L; ++i) mapping[i] = i;
    for (int i = L - 1; i > 0; --i) {
        const int j = static_cast<int>(rng.next_below(static_cast<uint64_t>(i) + 1));
        std::swap(mapping[i], mapping[j]);
    }
}

// engine.cpp:101-103: w0[i] = 0.1 * next_gaussian() from stream 0xA001.
void ref_init_w0(uint64_t seed, int64_t D, double* w0) {
    adpsgd::Rng r(adpsgd::derive_seed(seed, 0xA001));
    for (int64_t i = 0; i < D; ++i) w0[i] = 0.1 * r.next_gaussian();
}

// engine.cpp:112 + objectives.cpp:244-247: learner stream 0xB000+l, M draws per step.
void ref_learner_batches(uint64_t seed, int learner, int n_steps, int M, int train_count, int32_t* out) {
    adpsgd::Rng r(adpsgd::derive_seed(seed, 0xB000 + static_cast<uint64_t>(learner)));
    for (int64_t i = 0; i < static_cast<int64_t>(n_steps) * M; ++i)
        out[i] = static_cast<int32_t>(r.next_below(static_cast<uint64_t>(train_count)));
}

}
