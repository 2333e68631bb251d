// Cross-GPU transport for one-process-per-GPU runs: NCCL (dlopen'ed, shares the
// process's libnccl.so.2) for allreduce / barrier / send-recv, CUDA IPC for direct
// NVLink peer reads of neighbour weights.
#pragma once

#include <cuda_runtime.h>

#include <map>
#include <vector>

#include "common.cuh"

namespace ab {

struct Ctx;

class Comm {
  public:
    Comm(Ctx& ctx, int rank, int world, const void* nccl_id128);
    // single-process group transport (adpsgd_group_link): no NCCL, no IPC -- the other contexts'
    // buffers are read in place (cudaDeviceEnablePeerAccess across devices)
    struct LocalGroupTag {};
    Comm(Ctx& ctx, int rank, int world, LocalGroupTag);
    bool local_group = false;
    std::vector<Ctx*> group_ctxs;
    void link_local(Ctx& peer);
    const float* peer_grad(int gid) const;
    ~Comm();
    static void unique_id(void* out128);

    int rank = 0, world = 1;
    bool ipc_only = false;  // no NCCL (ranks sharing one GPU): FM/RM peer gossip, host-separated steps
    int gossip_mode = 0;  // 0 direct peer loads, 1 copy-engine prefetch, 2 NCCL send/recv
    // ADPSGD_COMM_FORCE=1 with a world-1 NCCL communicator: take every multi-rank branch (device
    // barrier, D1D weight allreduce overlapped with the compute, SDPSGD gradient allreduce, NCCL
    // send/recv gossip as self exchanges) so those call sites run, and are checked, on one GPU
    bool forced = false;
    bool multi() const { return world > 1 || forced; }
    // device-time stamps (ms after the step's start event) of the last D1D weight allreduce
    cudaEvent_t t_ar0 = nullptr, t_ar1 = nullptr;
    bool ar_pending = false;  // a D1D weight allreduce was issued this step (t_ar0 / t_ar1 valid)

    // SDPSGD: sum of every learner's gradient (in place in a comm buffer).
    const float* allreduce_sum_grads(Ctx& c, cudaStream_t s);
    // D1D: allreduce of w_k launched on the comm stream before the gradient compute ...
    void start_weight_sum(Ctx& c, cudaStream_t s);
    // ... and joined before the update.
    const float* wait_weight_sum(Ctx& c, cudaStream_t s);
    // FM/RM: GPU-side barrier so that every neighbour's w_k is final before the pulls.
    void pre_gossip(Ctx& c, cudaStream_t s);
    void barrier(cudaStream_t s);
    const float* peer_weight(int gid, int buf) const;
    const unsigned long long* peer_ver(int gid) const;  // publication counters (async FM/RM)
    // gossip_mode 1: copy-engine pulls of the two neighbours' w_k into local buffers on the comm
    // stream (issued at step start, overlapping the gradient compute; `ready` event joined by the mix)
    void prefetch_neighbours(Ctx& c, const float* wl, const float* wr, cudaStream_t s);
    // gossip_mode 2 (baseline): NCCL send of w_k to both neighbours / receive of theirs, on s
    void sendrecv_neighbours(Ctx& c, int j, int left, int right, cudaStream_t s);
    const float* nb_left() const { return nb_[0]; }
    const float* nb_right() const { return nb_[1]; }
    cudaEvent_t nb_ready = nullptr;

    int64_t ipc_size(const Ctx& c) const;
    static int64_t ipc_record_bytes();  // export bytes per local learner
    void export_ipc(const Ctx& c, void* out, int64_t size) const;
    void import_ipc(int peer_rank, int first, int count, const void* handles, int64_t size);

  private:
    void* nccl_ = nullptr;  // ncclComm_t
    float* wsum_ = nullptr;
    float* gsum_ = nullptr;
    float* bar_ = nullptr;
    cudaEvent_t ev_start_ = nullptr, ev_ws_ = nullptr;
    struct PeerMap {
        float* w[4] = {nullptr, nullptr, nullptr, nullptr};  // model versions (ring of nbuf)
        int nbuf = 0;
        unsigned long long* ver = nullptr;                   // publication counters
        const float* g = nullptr;                            // gradient (single-process group only)
    };
    std::map<int, PeerMap> peers_;  // gid -> that learner's buffers mapped over NVLink (CUDA IPC)
    std::vector<void*> opened_;
    float* nb_[2] = {nullptr, nullptr};  // local copies of the neighbours' w_k (modes 1, 2)
    void ensure_nb(Ctx& c);
    int64_t D_ = 0;
};

}  // namespace ab
