#include "knobs.hpp"

#include <cstdlib>

namespace ab {

namespace {
bool flag(const char* name, bool dflt, bool set_value) {
    const char* e = std::getenv(name);
    if (!e || !e[0]) return dflt;
    return e[0] == '1' ? set_value : (e[0] == '0' ? !set_value : dflt);
}
int num(const char* name) {
    const char* e = std::getenv(name);
    return e ? std::atoi(e) : 0;
}
Knobs load() {
    Knobs k;
    k.pair_mma = flag("ADPSGD_NO_PAIR", true, false);
    k.wide_fwd = flag("ADPSGD_NO_WIDE", true, false);
    k.splitk_bwd = flag("ADPSGD_NO_SPLITK", true, false);
    k.persist_fwd = flag("ADPSGD_NO_PERSIST_FWD", true, false);
    k.persist_bwd = flag("ADPSGD_NO_PERSIST", true, false);
    k.pdl = flag("ADPSGD_NO_PDL", true, false);
    k.streamk = flag("ADPSGD_NO_STREAMK", true, false);
    k.xtra = flag("ADPSGD_NO_XTRA", true, false);
    k.wide_gemm = flag("ADPSGD_NO_WIDE_GEMM", true, false);
    k.graphs = flag("ADPSGD_NO_GRAPHS", true, false);
    k.fused_cell = flag("ADPSGD_NO_FUSED", true, false);
    k.fold_bias = flag("ADPSGD_NO_FOLD_BIAS", true, false);
    k.fold_ih = flag("ADPSGD_NO_FOLD_IH", true, false);
    k.fwd_u32 = flag("ADPSGD_NO_FWD_U32", true, false);
    k.bwd_u32 = flag("ADPSGD_NO_BWD_U32", true, false);
    k.bwd_kmajor = flag("ADPSGD_BWD_KMAJOR", false, true);
    k.no_tma3d = flag("ADPSGD_NO_TMA3D", false, true);
    k.unfused_ce = flag("ADPSGD_UNFUSED_CE", false, true);
    k.fused_update = flag("ADPSGD_FUSED_UPDATE", false, true);
    k.bwd_kq4 = flag("ADPSGD_BWD_KQ4", false, true);
    k.wide_wgrad = flag("ADPSGD_WIDE_WGRAD", false, true);
    k.mcb = flag("ADPSGD_MCB", false, true);
    k.force_ext = flag("ADPSGD_FORCE_EXT", false, true);
    k.force_bn = num("ADPSGD_FORCE_BN");
    k.epi_skip = num("ADPSGD_EPI_SKIP");
    k.export_dbg = num("ADPSGD_EXPORT_DBG");
    k.async_hold_ms = num("ADPSGD_ASYNC_HOLD_MS");
    k.comm_force = flag("ADPSGD_COMM_FORCE", false, true);
    k.fwd_l2win = flag("ADPSGD_FWD_L2WIN", false, true);
    if (std::getenv("ADPSGD_PITCH_ALIGN")) k.pitch_align = num("ADPSGD_PITCH_ALIGN");
    if (std::getenv("ADPSGD_POISON_ALLOC")) k.poison_alloc = num("ADPSGD_POISON_ALLOC");
    if (std::getenv("ADPSGD_SPLIT_MAX")) k.split_max = num("ADPSGD_SPLIT_MAX");
    return k;
}

Knobs g_knobs = load();
}  // namespace

// The engine re-reads the environment at every context creation (tests flip switches between
// contexts); the kernels read the snapshot.
const Knobs& knobs() { return g_knobs; }
void reload_knobs() { g_knobs = load(); }

}  // namespace ab
