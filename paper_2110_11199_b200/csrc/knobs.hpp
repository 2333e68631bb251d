// Process-wide tuning / experiment switches, read once from the environment (knobs.cu).
// Defaults are the measured-best configuration; every switch is documented in DESIGN.md §4a.
#pragma once

namespace ab {

struct Knobs {
    // kernel selection (defaults on)
    bool pair_mma = true;      // ADPSGD_NO_PAIR=1: single-CTA tcgen05 tiles instead of CTA pairs
    bool wide_fwd = true;      // ADPSGD_NO_WIDE=1: per-step forward without 256x512 one-wave tiles
    bool splitk_bwd = true;    // ADPSGD_NO_SPLITK=1: per-step BPTT without the split-K variant
    bool persist_fwd = true;   // ADPSGD_NO_PERSIST_FWD=1: per-step forward launches
    bool persist_bwd = true;   // ADPSGD_NO_PERSIST=1: per-step BPTT launches
    bool pdl = true;           // ADPSGD_NO_PDL=1: no programmatic dependent launch
    bool streamk = true;       // ADPSGD_NO_STREAMK=1: no stream-K GEMMs
    bool xtra = true;          // ADPSGD_NO_XTRA=1: no extra row-sum MMA for bias columns
    bool wide_gemm = true;     // ADPSGD_NO_WIDE_GEMM=1: no 256x512 generic GEMM tiles
    bool graphs = true;        // ADPSGD_NO_GRAPHS=1: eager launches instead of CUDA graphs
    bool fused_cell = true;    // ADPSGD_NO_FUSED=1: unfused GEMM + pointwise LSTM cell
    bool fold_bias = true;     // ADPSGD_NO_FOLD_BIAS=1: bias gradients by column sums
    bool fold_ih = true;       // ADPSGD_NO_FOLD_IH=1: dW_ih bias gradients by column sums
    // measured slower, kept opt-in
    bool bwd_kq4 = false;      // ADPSGD_BWD_KQ4=1: persistent BPTT in K quarters
    bool wide_wgrad = false;   // ADPSGD_WIDE_WGRAD=1: one-wave 512-wide weight gradients
    bool mcb = false;          // ADPSGD_MCB=1: B operand TMA-multicast across two CTA pairs
    bool fused_update = false; // ADPSGD_FUSED_UPDATE=1: single learner's SGD update in the weight-gradient epilogues
    // tests / diagnosis
    bool force_ext = false;    // ADPSGD_FORCE_EXT=1: take the extra-column / stream-K / wide kernels wherever legal
    int force_bn = 0;          // ADPSGD_FORCE_BN=128|256: generic GEMM tile width (probes)
    int epi_skip = 0;          // ADPSGD_EPI_SKIP=n: epilogue timing experiments
    int export_dbg = 0;        // ADPSGD_EXPORT_DBG=1|2: split-K export diagnosis
    bool comm_force = false;   // ADPSGD_COMM_FORCE=1: a world-1 NCCL communicator takes the multi-rank branches (tests)
    int async_hold_ms = 0;     // ADPSGD_ASYNC_HOLD_MS=n: device delay between the first async mix and its torn-read check (tests the retry path)
    int split_max = 4;         // ADPSGD_SPLIT_MAX=n: K slices of the one-wave split-K weight gradients (1: off)
    bool fwd_u32 = true;       // ADPSGD_NO_FWD_U32=1: persistent forward always in 64-unit tiles
    bool bwd_u32 = true;       // ADPSGD_NO_BWD_U32=1: persistent BPTT always with 64 units per CTA
    bool no_tma3d = false;     // ADPSGD_NO_TMA3D=1: MN-major GEMM operands as two 2-D boxes per k-block (no 3-D views)
    bool bwd_kmajor = false;   // ADPSGD_BWD_KMAJOR=1: 64-unit persistent BPTT reads a K-major W_hh^T (else MN-major W_hh)
    int pitch_align = 64;      // ADPSGD_PITCH_ALIGN=n: activation row pitches (elements) rounded up to n (1: unpadded)
    bool fwd_l2win = false;    // ADPSGD_FWD_L2WIN=1: persisting L2 window over the persistent forward's weights
    int poison_alloc = -1;     // ADPSGD_POISON_ALLOC=b: fill every engine allocation with byte b (0xFF = NaN) -- initcheck triage
    bool unfused_ce = false;   // ADPSGD_UNFUSED_CE=1: bf16 logits GEMM (fp32 out) + softmax-CE kernel (diagnosis)
};

const Knobs& knobs();
void reload_knobs();  // re-read the environment (engine context creation)

}  // namespace ab
