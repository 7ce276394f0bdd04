// dvm_peer.cu -- direction-shard reduction over peer memory (sm_100a, fp64).
//
// Q = Σ_e Q_e is a sum over the directions (eq:decD) and the
// directions are split over the ranks ("completely
// parallelizable"), so Q = Σ_r Q_r.  Instead of a separate NCCL all-reduce the
// partial is pushed once into every rank's peer window over NVLink (P2P
// stores, one-shot), and every rank adds the W slots of its own window in rank
// order: no reduction tree, identical bits on every rank, the transfer of one
// CTA's chunk overlapping the others' (see include/dvm.h for the layout).
//
//   k_peer_push:   grid-stride over the partial (double2), every CTA writes its
//                  chunk into slot `rank` of each peer window, then one thread
//                  fences at system scope (cumulative over the CTA barrier) and
//                  adds 1 to counter `rank` of every window.
//   k_peer_reduce: thread 0 of each CTA waits (acquire, system scope) until all
//                  W counters reach epoch × push CTAs, then the CTA sums its
//                  elements over the slots in rank order.
// The push grid is a function of the element count only, so every rank
// expects the same number of arrivals.
#include <stdint.h>
#include <string.h>

#include "dvm_internal.h"

namespace dvm {
namespace {

constexpr int kPeerThreads = 256;
constexpr int kMaxWorld = 64;

struct PeerPtrs {
    double2 *slot[kMaxWorld];       // slot `rank` of window r (as mapped here)
    unsigned int *ctr[kMaxWorld];   // counter `rank` of window r
};

int64_t nodes_per_cell(const dvm_plan_s *P)
{
    int64_t n = 1;
    for (int j = 0; j < P->d; ++j) n *= P->N;
    return n;
}

// push CTAs for n doubles (n even: N^d with N a power of two >= 4)
int push_blocks(int64_t n)
{
    const int64_t b = (n / 2 + kPeerThreads - 1) / kPeerThreads;
    return (int)(b < 1184 ? (b < 1 ? 1 : b) : 1184);  // 8 CTAs per SM of 148
}

size_t slots_bytes(int64_t n, int world)
{
    // counters start 256-byte aligned after the slots
    return ((size_t)world * (size_t)n * sizeof(double) + 255) & ~(size_t)255;
}

__global__ void __launch_bounds__(kPeerThreads) k_peer_push(const double2 *__restrict__ part, int64_t n2,
                                                             PeerPtrs peers, int world, int rank)
{
    for (int64_t i = (int64_t)blockIdx.x * kPeerThreads + threadIdx.x; i < n2;
         i += (int64_t)gridDim.x * kPeerThreads) {
        const double2 v = part[i];
        for (int r = 0; r < world; ++r)
            if (r != rank) peers.slot[r][i] = v;  // P2P store over NVLink (the local slot holds v already)
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        // every thread's stores of this CTA are ordered before the arrivals
        // (bar.sync + fence.sc.sys is cumulative)
        asm volatile("fence.sc.sys;" ::: "memory");
        for (int r = 0; r < world; ++r) asm volatile("red.release.sys.global.add.u32 [%0], 1;" ::"l"(peers.ctr[r]) : "memory");
    }
}

__global__ void __launch_bounds__(kPeerThreads) k_peer_reduce(const double2 *__restrict__ slots,
                                                               const unsigned int *ctr, double2 *__restrict__ Q,
                                                               int64_t n2, int world, unsigned int target)
{
    if (threadIdx.x == 0) {
        for (int r = 0; r < world; ++r) {
            unsigned int v;
            for (;;) {
                asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr + r) : "memory");
                if ((int)(v - target) >= 0) break;
                __nanosleep(64);
            }
        }
    }
    __syncthreads();
    for (int64_t i = (int64_t)blockIdx.x * kPeerThreads + threadIdx.x; i < n2;
         i += (int64_t)gridDim.x * kPeerThreads) {
        double2 s = __ldcv(&slots[i]);  // slot 0 (written by a peer: bypass L1)
        for (int r = 1; r < world; ++r) {
            const double2 v = __ldcv(&slots[(int64_t)r * n2 + i]);
            s.x += v.x;
            s.y += v.y;
        }
        Q[i] = s;
    }
}

dvm_status_t check_peer(dvm_plan_s *P, int64_t ncells, int world)
{
    if (!P) {
        set_error("NULL plan");
        return DVM_E_NULL;
    }
    if (ncells < 1 || world < 1 || world > kMaxWorld) {
        set_error("peer window: ncells >= 1 and 1 <= world <= 64");
        return DVM_E_SHAPE;
    }
    if (world != P->shard_world) {
        set_error("peer window: world must equal the plan's shard_world");
        return DVM_E_STATE;
    }
    return DVM_OK;
}

}  // namespace

dvm_status_t peer_push_check(dvm_plan_s *P, const double *f, int64_t ncells, void *const *windows, int rank,
                             int world, unsigned int epoch, double **mine)
{
    if (!P || !f || !windows) {
        set_error("NULL argument");
        return DVM_E_NULL;
    }
    dvm_status_t st = check_peer(P, ncells, world);
    if (st) return st;
    if (rank != P->shard_rank || epoch == 0) {
        set_error(epoch == 0 ? "epoch must be >= 1" : "rank must equal the plan's shard_rank");
        return DVM_E_STATE;
    }
    for (int r = 0; r < world; ++r)
        if (!windows[r]) {
            set_error("NULL peer window");
            return DVM_E_NULL;
        }
    *mine = (double *)windows[rank] + (size_t)rank * (size_t)(ncells * nodes_per_cell(P));
    return DVM_OK;
}

dvm_status_t peer_push_launch(dvm_plan_s *P, const double *mine, int64_t n, void *const *windows, int rank,
                              int world)
{
    const size_t cofs = slots_bytes(n, world);
    PeerPtrs pp;
    for (int r = 0; r < world; ++r) {
        pp.slot[r] = (double2 *)((double *)windows[r] + (size_t)rank * n);
        pp.ctr[r] = (unsigned int *)((char *)windows[r] + cofs) + rank;
    }
    {
        LaunchScope ls(P, KC_REDUCE);
        k_peer_push<<<push_blocks(n), kPeerThreads, 0, P->stream>>>((const double2 *)mine, n / 2, pp, world, rank);
    }
    DVM_CUDA(cudaGetLastError());
    return DVM_OK;
}

}  // namespace dvm

using namespace dvm;

extern "C" {

size_t dvm_peer_window_bytes(dvm_plan_t P, int64_t ncells, int world)
{
    if (!P || ncells < 1 || world < 1 || world > kMaxWorld) return 0;
    return slots_bytes(ncells * nodes_per_cell(P), world) + sizeof(unsigned int) * (size_t)world;
}

dvm_status_t dvm_peer_window_alloc(dvm_plan_t P, int64_t ncells, int world, void **out)
{
    if (!out) {
        set_error("NULL argument");
        return DVM_E_NULL;
    }
    *out = nullptr;
    dvm_status_t st = check_peer(P, ncells, world);
    if (st) return st;
    DVM_CUDA(cudaSetDevice(P->device));
    const size_t bytes = dvm_peer_window_bytes(P, ncells, world);
    void *w = nullptr;
    if (cudaMalloc(&w, bytes) != cudaSuccess) {
        cudaGetLastError();
        set_error("peer window allocation failed");
        return DVM_E_NOMEM;
    }
    const size_t off = slots_bytes(ncells * nodes_per_cell(P), world);
    DVM_CUDA(cudaMemset((char *)w + off, 0, bytes - off));
    *out = w;
    return DVM_OK;
}

dvm_status_t dvm_peer_window_free(void *w)
{
    if (w) DVM_CUDA(cudaFree(w));
    return DVM_OK;
}

dvm_status_t dvm_ipc_handle(const void *dptr, unsigned char handle[64])
{
    if (!dptr || !handle) {
        set_error("NULL argument");
        return DVM_E_NULL;
    }
    static_assert(sizeof(cudaIpcMemHandle_t) == 64, "CUDA IPC handles are 64 bytes");
    cudaIpcMemHandle_t h;
    DVM_CUDA(cudaIpcGetMemHandle(&h, const_cast<void *>(dptr)));
    memcpy(handle, &h, 64);
    return DVM_OK;
}

dvm_status_t dvm_ipc_open(const unsigned char handle[64], void **out)
{
    if (!handle || !out) {
        set_error("NULL argument");
        return DVM_E_NULL;
    }
    cudaIpcMemHandle_t h;
    memcpy(&h, handle, 64);
    DVM_CUDA(cudaIpcOpenMemHandle(out, h, cudaIpcMemLazyEnablePeerAccess));
    return DVM_OK;
}

dvm_status_t dvm_ipc_close(void *dptr)
{
    if (dptr) DVM_CUDA(cudaIpcCloseMemHandle(dptr));
    return DVM_OK;
}

dvm_status_t dvm_peer_reduce(dvm_plan_t P, const void *window, double *Q, int64_t ncells, int world,
                             unsigned int epoch)
{
    if (!P || !window || !Q) {
        set_error("NULL argument");
        return DVM_E_NULL;
    }
    dvm_status_t st = check_peer(P, ncells, world);
    if (st) return st;
    if (epoch == 0) {
        set_error("epoch must be >= 1");
        return DVM_E_STATE;
    }
    const int64_t n = ncells * nodes_per_cell(P);
    const unsigned int target = epoch * (unsigned int)push_blocks(n);
    const unsigned int *ctr = (const unsigned int *)((const char *)window + slots_bytes(n, world));
    {
        LaunchScope ls(P, KC_REDUCE);
        // at most one CTA per SM waits: every CTA spins only on its own thread 0
        const int blocks = push_blocks(n) < 148 ? push_blocks(n) : 148;
        k_peer_reduce<<<blocks, kPeerThreads, 0, P->stream>>>((const double2 *)window, ctr, (double2 *)Q, n / 2,
                                                               world, target);
    }
    DVM_CUDA(cudaGetLastError());
    return DVM_OK;
}

}  // extern "C"
