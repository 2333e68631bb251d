// NCCL + CUDA-IPC transport (see comm.hpp). NCCL is resolved with dlopen so the
// library shares whichever libnccl.so.2 the process already loaded (torch's).
#include "comm.hpp"

#include <cstdlib>

#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>
#include <string>

#include "engine.hpp"
#include "kernels.cuh"
#include "knobs.hpp"

namespace ab {

namespace {

struct NcclApi {
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi& nccl() {
    static NcclApi api;
    static std::once_flag once;
    static std::string err;
    std::call_once(once, [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) { err = dlerror() ? dlerror() : "dlopen libnccl failed"; return; }
        api.GetUniqueId = reinterpret_cast<decltype(api.GetUniqueId)>(dlsym(h, "ncclGetUniqueId"));
        api.CommInitRank = reinterpret_cast<decltype(api.CommInitRank)>(dlsym(h, "ncclCommInitRank"));
        api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(dlsym(h, "ncclCommDestroy"));
        api.AllReduce = reinterpret_cast<decltype(api.AllReduce)>(dlsym(h, "ncclAllReduce"));
        api.Send = reinterpret_cast<decltype(api.Send)>(dlsym(h, "ncclSend"));
        api.Recv = reinterpret_cast<decltype(api.Recv)>(dlsym(h, "ncclRecv"));
        api.GroupStart = reinterpret_cast<decltype(api.GroupStart)>(dlsym(h, "ncclGroupStart"));
        api.GroupEnd = reinterpret_cast<decltype(api.GroupEnd)>(dlsym(h, "ncclGroupEnd"));
        api.GetErrorString = reinterpret_cast<decltype(api.GetErrorString)>(dlsym(h, "ncclGetErrorString"));
    });
    AB_CHECK(api.AllReduce && api.CommInitRank, ADPSGD_E_NCCL, "NCCL unavailable: " + err);
    return api;
}

#define AB_NCCL(x)                                                                                     \
    do {                                                                                               \
        ncclResult_t r_ = (x);                                                                         \
        if (r_ != ncclSuccess)                                                                         \
            throw ::ab::Error(ADPSGD_E_NCCL, std::string(#x) + ": " +                                  \
                                                 (nccl().GetErrorString ? nccl().GetErrorString(r_) : "")); \
    } while (0)

constexpr int kHandle = static_cast<int>(sizeof(cudaIpcMemHandle_t));

}  // namespace

void Comm::unique_id(void* out128) {
    ncclUniqueId id;
    AB_NCCL(nccl().GetUniqueId(&id));
    std::memcpy(out128, &id, sizeof(id));
}

Comm::Comm(Ctx& c, int r, int w, const void* id128) : rank(r), world(w), D_(c.D) {
    AB_CHECK(w >= 1 && r >= 0 && r < w, ADPSGD_E_CONFIG, "bad rank/world");
    AB_CHECK(w == 1 || c.cfg.local_learners == 1, ADPSGD_E_CONFIG,
             "multi-process runs host exactly one learner per rank");
    if (id128 == nullptr) {
        // CUDA-IPC-only transport: FM/RM pulls from peer buffers; the caller separates steps with
        // a host barrier (there is no device barrier). For ranks sharing one GPU, where NCCL
        // refuses duplicate devices -- tests of the multi-process gossip path on one B200.
        ipc_only = true;
        return;
    }
    forced = w == 1 && knobs().comm_force;
    // The D1D weight allreduce runs concurrently with the persistent recurrent kernels, which need
    // all their 2 x 64 CTAs co-resident (cross-CTA step counters) and leave 148 - 128 = 20 SMs free:
    // cap NCCL's CTAs so its kernel fits beside them instead of holding SMs the forward is waiting
    // for (16 CTAs move the 0.58 GB allreduce well inside the forward). A user setting wins.
    if (!std::getenv("NCCL_MAX_CTAS")) setenv("NCCL_MAX_CTAS", "16", 0);
    ncclUniqueId id;
    std::memcpy(&id, id128, sizeof(id));
    ncclComm_t comm;
    AB_NCCL(nccl().CommInitRank(&comm, w, id, r));
    nccl_ = comm;
    wsum_ = static_cast<float*>(c.alloc(c.D * sizeof(float)));
    gsum_ = static_cast<float*>(c.alloc(c.D * sizeof(float)));
    bar_ = static_cast<float*>(c.alloc(sizeof(float) * 4));
    AB_CUDA(cudaMemsetAsync(bar_, 0, sizeof(float) * 4, c.s_main));
    AB_CUDA(cudaStreamSynchronize(c.s_main));
    AB_CUDA(cudaEventCreateWithFlags(&ev_start_, cudaEventDisableTiming));
    AB_CUDA(cudaEventCreateWithFlags(&ev_ws_, cudaEventDisableTiming));
    AB_CUDA(cudaEventCreate(&t_ar0));
    AB_CUDA(cudaEventCreate(&t_ar1));
}

Comm::Comm(Ctx& c, int r, int w, LocalGroupTag) : rank(r), world(w), D_(c.D) {
    AB_CHECK(w >= 1 && r >= 0 && r < w, ADPSGD_E_CONFIG, "bad group rank/size");
    ipc_only = true;  // the host joins every context at the end of each group step
    local_group = true;
}

// Map a linked context's learners into this one: weights, publication counters and gradients are
// read in place (same process; P2P over NVLink when the devices differ).
void Comm::link_local(Ctx& peer) {
    for (const Learner& ln : peer.learners) {
        PeerMap pm;
        pm.nbuf = peer.nbuf;
        for (int b = 0; b < peer.nbuf; ++b) pm.w[b] = ln.w[b];
        pm.ver = ln.ver;
        pm.g = ln.g;
        peers_[ln.gid] = pm;
    }
}

const float* Comm::peer_grad(int gid) const {
    auto it = peers_.find(gid);
    AB_CHECK(it != peers_.end() && it->second.g, ADPSGD_E_INVALID_STATE,
             "learner " + std::to_string(gid) + "'s gradient is not mapped (single-process groups only)");
    return it->second.g;
}

void Comm::ensure_nb(Ctx& c) {
    if (!nb_[0]) {
        nb_[0] = static_cast<float*>(c.alloc(c.D * sizeof(float)));
        nb_[1] = static_cast<float*>(c.alloc(c.D * sizeof(float)));
        AB_CUDA(cudaEventCreateWithFlags(&nb_ready, cudaEventDisableTiming));
    }
}

void Comm::prefetch_neighbours(Ctx& c, const float* wl, const float* wr, cudaStream_t s) {
    ensure_nb(c);
    // (NCCL transport: every rank's w_k is final once the barrier on s has completed)
    barrier(s);
    AB_CUDA(cudaEventRecord(nb_ready, s));
    AB_CUDA(cudaStreamWaitEvent(c.s_comm, nb_ready, 0));
    AB_CUDA(cudaMemcpyAsync(nb_[0], wl, c.D * sizeof(float), cudaMemcpyDeviceToDevice, c.s_comm));
    AB_CUDA(cudaMemcpyAsync(nb_[1], wr, c.D * sizeof(float), cudaMemcpyDeviceToDevice, c.s_comm));
    AB_CUDA(cudaEventRecord(nb_ready, c.s_comm));
}

void Comm::sendrecv_neighbours(Ctx& c, int j, int left, int right, cudaStream_t s) {
    AB_CHECK(!ipc_only, ADPSGD_E_CONFIG, "gossip mode 2 (NCCL send/recv) needs the NCCL transport");
    ensure_nb(c);
    auto* comm = static_cast<ncclComm_t>(nccl_);
    if (world == 1) {
        // forced single-rank mode: every neighbour is local -- each one's w_k goes through an NCCL
        // send / recv pair with this rank itself
        AB_NCCL(nccl().GroupStart());
        AB_NCCL(nccl().Send(c.weight_ptr(left, c.slot(c.k)), c.D, ncclFloat32, 0, comm, s));
        AB_NCCL(nccl().Send(c.weight_ptr(right, c.slot(c.k)), c.D, ncclFloat32, 0, comm, s));
        AB_NCCL(nccl().Recv(nb_[0], c.D, ncclFloat32, 0, comm, s));
        AB_NCCL(nccl().Recv(nb_[1], c.D, ncclFloat32, 0, comm, s));
        AB_NCCL(nccl().GroupEnd());
        return;
    }
    AB_CHECK(c.cfg.local_learners == 1 && j == 0, ADPSGD_E_CONFIG, "NCCL send/recv gossip hosts one learner per rank");
    const float* w = c.learners[0].w[c.slot(c.k)];
    const int rl = left - c.cfg.first_learner + rank, rr = right - c.cfg.first_learner + rank;  // one learner per rank
    AB_NCCL(nccl().GroupStart());
    AB_NCCL(nccl().Send(w, c.D, ncclFloat32, rl, comm, s));
    AB_NCCL(nccl().Send(w, c.D, ncclFloat32, rr, comm, s));
    AB_NCCL(nccl().Recv(nb_[0], c.D, ncclFloat32, rl, comm, s));
    AB_NCCL(nccl().Recv(nb_[1], c.D, ncclFloat32, rr, comm, s));
    AB_NCCL(nccl().GroupEnd());
}

Comm::~Comm() {
    if (nb_ready) cudaEventDestroy(nb_ready);
    for (void* p : opened_) cudaIpcCloseMemHandle(p);
    if (nccl_) nccl().CommDestroy(static_cast<ncclComm_t>(nccl_));
    if (ev_start_) cudaEventDestroy(ev_start_);
    if (ev_ws_) cudaEventDestroy(ev_ws_);
    if (t_ar0) cudaEventDestroy(t_ar0);
    if (t_ar1) cudaEventDestroy(t_ar1);
}

void Comm::barrier(cudaStream_t s) {
    if (ipc_only) return;  // steps are separated on the host
    AB_NCCL(nccl().AllReduce(bar_, bar_ + 1, 1, ncclFloat32, ncclSum, static_cast<ncclComm_t>(nccl_), s));
}

// Local learners' contribution in learner order (the single-process kernels' summation order),
// then the sum over ranks in place.
static const float* local_sum(Ctx& c, bool grads, float* buf, cudaStream_t s) {
    if (c.cfg.local_learners == 1) return grads ? c.learners[0].g : c.learners[0].w[c.slot(c.k)];
    std::vector<const float*> tab;
    for (auto& ln : c.learners) tab.push_back(grads ? ln.g : ln.w[c.slot(c.k)]);
    launch_sum_tab(c.D, static_cast<int>(tab.size()), tab.data(), buf, s);
    return buf;
}

const float* Comm::allreduce_sum_grads(Ctx& c, cudaStream_t s) {
    AB_CHECK(!ipc_only, ADPSGD_E_CONFIG, "IPC-only transport: FM / RM only (SDPSGD needs NCCL)");
    const float* src = local_sum(c, true, gsum_, s);
    AB_NCCL(nccl().AllReduce(src, gsum_, c.D, ncclFloat32, ncclSum, static_cast<ncclComm_t>(nccl_), s));
    return gsum_;
}

void Comm::start_weight_sum(Ctx& c, cudaStream_t s) {
    AB_CHECK(!ipc_only, ADPSGD_E_CONFIG, "IPC-only transport: FM / RM only (D1D needs NCCL)");
    // w_k is final once the previous iteration's update (enqueued on s) has run.
    AB_CUDA(cudaEventRecord(ev_start_, s));
    AB_CUDA(cudaStreamWaitEvent(c.s_comm, ev_start_, 0));
    AB_CUDA(cudaEventRecord(t_ar0, c.s_comm));
    const float* src = local_sum(c, false, wsum_, c.s_comm);
    AB_NCCL(nccl().AllReduce(src, wsum_, c.D, ncclFloat32, ncclSum, static_cast<ncclComm_t>(nccl_), c.s_comm));
    AB_CUDA(cudaEventRecord(t_ar1, c.s_comm));
    AB_CUDA(cudaEventRecord(ev_ws_, c.s_comm));
    ar_pending = true;
}

const float* Comm::wait_weight_sum(Ctx& c, cudaStream_t s) {
    (void)c;
    AB_CUDA(cudaStreamWaitEvent(s, ev_ws_, 0));
    return wsum_;
}

void Comm::pre_gossip(Ctx& c, cudaStream_t s) {
    (void)c;
    barrier(s);
}

const float* Comm::peer_weight(int gid, int buf) const {
    auto it = peers_.find(gid);
    AB_CHECK(it != peers_.end(), ADPSGD_E_INVALID_STATE,
             "learner " + std::to_string(gid) + " has no mapped weights (adpsgd_import_ipc)");
    AB_CHECK(buf >= 0 && buf < it->second.nbuf, ADPSGD_E_INVALID_STATE,
             "learner " + std::to_string(gid) + " exports " + std::to_string(it->second.nbuf) +
                 " model versions (async rings must be enabled on every rank before export)");
    return it->second.w[buf];
}

const unsigned long long* Comm::peer_ver(int gid) const {
    auto it = peers_.find(gid);
    AB_CHECK(it != peers_.end() && it->second.ver, ADPSGD_E_INVALID_STATE,
             "learner " + std::to_string(gid) + " has no mapped publication counters (adpsgd_import_ipc)");
    return it->second.ver;
}

// Export record per local learner: int32 nbuf, int32 reserved, then 4 weight-slot handles (the
// first nbuf valid) and the publication-counter handle.
namespace {
constexpr int kRec = 8 + 5 * kHandle;
}

int64_t Comm::ipc_record_bytes() { return kRec; }
int64_t Comm::ipc_size(const Ctx& c) const { return static_cast<int64_t>(c.cfg.local_learners) * kRec; }

void Comm::export_ipc(const Ctx& c, void* out, int64_t size) const {
    AB_CHECK(size >= ipc_size(c), ADPSGD_E_DIMENSION, "ipc buffer too small");
    uint8_t* o = static_cast<uint8_t*>(out);
    std::memset(o, 0, static_cast<size_t>(ipc_size(c)));
    for (int j = 0; j < c.cfg.local_learners; ++j) {
        uint8_t* r = o + static_cast<int64_t>(j) * kRec;
        const int32_t hdr[2] = {c.nbuf, 0};
        std::memcpy(r, hdr, sizeof(hdr));
        for (int b = 0; b < c.nbuf; ++b) {
            cudaIpcMemHandle_t h;
            AB_CUDA(cudaIpcGetMemHandle(&h, c.learners[j].w[b]));
            std::memcpy(r + 8 + b * kHandle, &h, kHandle);
        }
        cudaIpcMemHandle_t h;
        AB_CUDA(cudaIpcGetMemHandle(&h, c.learners[j].ver));
        std::memcpy(r + 8 + 4 * kHandle, &h, kHandle);
    }
}

void Comm::import_ipc(int peer_rank, int first, int count, const void* handles, int64_t size) {
    AB_CHECK(size >= static_cast<int64_t>(count) * kRec, ADPSGD_E_DIMENSION, "ipc buffer too small");
    if (peer_rank == rank) return;
    const uint8_t* in = static_cast<const uint8_t*>(handles);
    auto open = [&](const uint8_t* src) {
        cudaIpcMemHandle_t h;
        std::memcpy(&h, src, kHandle);
        void* ptr = nullptr;
        AB_CUDA(cudaIpcOpenMemHandle(&ptr, h, cudaIpcMemLazyEnablePeerAccess));
        opened_.push_back(ptr);
        return ptr;
    };
    for (int j = 0; j < count; ++j) {
        const uint8_t* r = in + static_cast<int64_t>(j) * kRec;
        int32_t hdr[2];
        std::memcpy(hdr, r, sizeof(hdr));
        AB_CHECK(hdr[0] == 2 || hdr[0] == 4, ADPSGD_E_INVALID_STATE, "corrupt IPC export record");
        PeerMap pm;
        pm.nbuf = hdr[0];
        for (int b = 0; b < pm.nbuf; ++b) pm.w[b] = static_cast<float*>(open(r + 8 + b * kHandle));
        pm.ver = static_cast<unsigned long long*>(open(r + 8 + 4 * kHandle));
        peers_[first + j] = pm;
    }
}

}  // namespace ab
