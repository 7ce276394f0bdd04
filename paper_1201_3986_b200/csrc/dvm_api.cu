// dvm_api.cu -- the extern "C" entry points of libdvm (include/dvm.h):
// parameter validation, plan life cycle, host<->device staging, status codes.
#include <math.h>
#include <string.h>

#include <atomic>
#include <new>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "dvm_internal.h"

namespace dvm {

static thread_local std::string g_last_error;

void set_error(const std::string &msg) { g_last_error = msg; }

dvm_status_t cuda_fail(cudaError_t err, const char *what)
{
    g_last_error = std::string(what) + ": " + cudaGetErrorString(err);
    return DVM_E_CUDA;
}

}  // namespace dvm

using namespace dvm;

namespace {
// NVTX range around every public entry point that launches work (header-only
// NVTX3: a no-op unless a profiler injects itself)
struct NvtxRange {
    explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
};
}  // namespace

namespace {

bool is_pow2(int n) { return n > 0 && (n & (n - 1)) == 0; }

dvm_status_t validate(const dvm_plan_params_t *p, int *Ntilde_out, double *L_out)
{
    if (p->d != 2 && p->d != 3) {
        set_error("d must be 2 or 3");
        return DVM_E_DIM;
    }
    if ((p->d == 2 && p->kernel != DVM_MAXWELL_2D) || (p->d == 3 && p->kernel != DVM_HARD_SPHERES_3D)) {
        set_error("kernel does not match d (2D Maxwell molecules, 3D hard spheres)");
        return DVM_E_KERNEL;
    }
    const int maxN = p->d == 2 ? 1024 : 256;
    if (!is_pow2(p->N) || p->N < 4 || p->N > maxN) {
        set_error("N must be a power of two in [4, 1024] (2D) / [4, 256] (3D)");
        return DVM_E_UNSUPPORTED;
    }
    double L = p->L == 0.0 ? 8.0 : p->L;
    if (!(L > 0.0) || !isfinite(L)) {
        set_error("L must be positive and finite");
        return DVM_E_UNSUPPORTED;
    }
    int Nt = p->Ntilde;
    if (Nt == 0) {  // reading R2: max(floor(N/(3+sqrt 2)), N̄)
        Nt = (int)floor((double)p->N / (3.0 + sqrt(2.0)));
        if (Nt < p->Nbar) Nt = p->Nbar;
    }
    if (p->Nbar < 1 || p->Nbar > Nt || 2 * Nt + 1 > p->N) {
        set_error("need 1 <= Nbar <= Ntilde and 2*Ntilde+1 <= N");
        return DVM_E_ORDER;
    }
    if (p->shard_world < 1 || p->shard_rank < 0 || p->shard_rank >= p->shard_world) {
        set_error("need 0 <= shard_rank < shard_world");
        return DVM_E_SHAPE;
    }
    *Ntilde_out = Nt;
    *L_out = L;
    return DVM_OK;
}

bool overlaps(const double *a, const double *b, int64_t n_a, int64_t n_b)
{
    const char *a0 = (const char *)a, *a1 = a0 + n_a * (int64_t)sizeof(double);
    const char *b0 = (const char *)b, *b1 = b0 + n_b * (int64_t)sizeof(double);
    return a0 < b1 && b0 < a1;
}

int64_t nodes_of(const dvm_plan_s *P)
{
    int64_t n = 1;
    for (int j = 0; j < P->d; ++j) n *= P->N;
    return n;
}

dvm_status_t check_batch(dvm_plan_s *P, const double *f, double *Q, int64_t ncells, int64_t *stride)
{
    if (!P || !f || !Q) {
        set_error("NULL argument");
        return DVM_E_NULL;
    }
    const int64_t nodes = nodes_of(P);
    if (*stride == 0) *stride = nodes;
    if (ncells < 0 || *stride < nodes || (ncells > 0 && *stride > (INT64_MAX / 8) / ncells)) {
        set_error("bad ncells / cell_stride");
        return DVM_E_SHAPE;
    }
    const int64_t span = ncells > 0 ? (ncells - 1) * *stride + nodes : 0;
    if (ncells > 0 && overlaps(f, Q, span, span)) {
        set_error("Q overlaps f");
        return DVM_E_ALIAS;
    }
    return DVM_OK;
}

}  // namespace

namespace dvm {
namespace {
std::atomic<uint64_t> g_ws_epoch{0};
}
uint64_t ws_epoch() { return g_ws_epoch.load(std::memory_order_relaxed); }
void ws_epoch_bump() { g_ws_epoch.fetch_add(1, std::memory_order_relaxed); }
}  // namespace dvm

namespace {
void drop_collide_graph(dvm_plan_s *P)
{
    if (P->cg.exec) cudaGraphExecDestroy(P->cg.exec);
    P->cg = dvm_plan_s::CollideGraph{};
}

// Capture work() (which issues everything on P->stream) on the plan's graph
// stream; true with cg.exec set if the whole call was capturable (any
// synchronising or allocating call inside fails the capture: the caller then
// runs it directly).
template <class Work>
bool capture_work(dvm_plan_s *P, Work &&work)
{
    if (!P->gstream) {
        if (cudaStreamCreateWithFlags(&P->gstream, cudaStreamNonBlocking) != cudaSuccess ||
            cudaEventCreateWithFlags(&P->gev[0], cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&P->gev[1], cudaEventDisableTiming) != cudaSuccess) {
            cudaGetLastError();
            return false;
        }
    }
    cudaStream_t user = P->stream;
    const uint64_t l0 = P->launches, e0 = ws_epoch();
    P->stream = P->gstream;
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    cudaError_t ce = cudaStreamBeginCapture(P->gstream, cudaStreamCaptureModeThreadLocal);
    dvm_status_t st = DVM_OK;
    if (ce == cudaSuccess) {
        st = work();
        ce = cudaStreamEndCapture(P->gstream, &graph);
        if (st == DVM_OK && ce == cudaSuccess && ws_epoch() == e0) ce = cudaGraphInstantiate(&exec, graph, 0);
    }
    P->stream = user;
    if (graph) cudaGraphDestroy(graph);
    const bool ok = st == DVM_OK && ce == cudaSuccess && exec && ws_epoch() == e0;
    if (!ok) {
        if (exec) cudaGraphExecDestroy(exec);
        cudaGetLastError();
        P->launches = l0;
        return false;
    }
    P->cg.exec = exec;
    P->cg.launches = P->launches - l0;
    P->launches = l0;
    return true;
}

// work() through the graph cache, keyed by (kind, a, b, n, stride) with the plan
// version and the workspace epoch: small batches are host-launch bound, so the
// second identical call is captured as one CUDA graph and later identical calls
// replay it (same kernels and copies, same bits)
template <class Work>
dvm_status_t run_cached(dvm_plan_s *P, int kind, const void *a, const void *b, int64_t ncells, int64_t cell_stride,
                        Work &&work)
{
    const bool small = ncells > 0 && (uint64_t)ncells * (uint64_t)nodes_of(P) <= (1ull << 22);
    // the persistent 3D gain kernels (N = 64; N = 32 beyond 2 cells or forced) rely
    // on a cooperative launch for co-residency of their CTA groups: never captured
    const bool coop = P->d == 3 && (P->N == 64 || (P->N == 32 && (ncells > 2 || (P->path_mode != 0 && P->path_mode != 6))));
    if (!P->use_graphs || P->profiling || !small || coop) return work();
    // a caller capturing its own graph on the plan's stream gets the plain launches
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(P->stream, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) {
        cudaGetLastError();
        return work();
    }
    auto &g = P->cg;
    const bool same = g.kind == kind && g.f == a && g.Q == b && g.n == ncells && g.stride == cell_stride &&
                      g.version == P->version && g.epoch == ws_epoch();
    if (same && g.state == 0) g.state = capture_work(P, work) ? 1 : 2;
    if (same && g.state == 1) {
        const cudaError_t ce = cudaGraphLaunch(g.exec, P->stream);
        if (ce == cudaSuccess) {
            P->launches += g.launches;
            return DVM_OK;
        }
        cudaGetLastError();
        drop_collide_graph(P);
        return work();
    }
    if (same) return work();  // capture failed for this key
    drop_collide_graph(P);
    const dvm_status_t st = work();
    g.kind = kind, g.f = a, g.Q = b, g.n = ncells, g.stride = cell_stride;
    g.version = P->version, g.epoch = ws_epoch(), g.state = 0;
    return st;
}
}  // namespace

extern "C" {

int dvm_abi_version(void) { return DVM_ABI_VERSION; }

const char *dvm_last_error(void) { return g_last_error.c_str(); }

const char *dvm_status_str(dvm_status_t s)
{
    switch (s) {
    case DVM_OK: return "DVM_OK";
    case DVM_E_NULL: return "DVM_E_NULL: NULL argument";
    case DVM_E_DIM: return "DVM_E_DIM: d must be 2 or 3";
    case DVM_E_KERNEL: return "DVM_E_KERNEL: kernel does not match d";
    case DVM_E_ORDER: return "DVM_E_ORDER: need 1 <= Nbar <= Ntilde, 2 Ntilde + 1 <= N";
    case DVM_E_UNSUPPORTED: return "DVM_E_UNSUPPORTED: unsupported N or L";
    case DVM_E_SHAPE: return "DVM_E_SHAPE: bad ncells, cell_stride or shard";
    case DVM_E_ALIAS: return "DVM_E_ALIAS: Q overlaps f";
    case DVM_E_NOMEM: return "DVM_E_NOMEM: allocation failed";
    case DVM_E_CUDA: return "DVM_E_CUDA: CUDA runtime error";
    case DVM_E_STATE: return "DVM_E_STATE: call not valid for this plan";
    }
    return "unknown dvm_status_t";
}

dvm_status_t dvm_plan_ex(const dvm_plan_params_t *params, dvm_plan_t *out)
{
    NvtxRange nvtx_range("dvm_plan_ex");
    if (!params || !out) {
        set_error("NULL argument");
        return DVM_E_NULL;
    }
    int Nt;
    double L;
    dvm_status_t st = validate(params, &Nt, &L);
    if (st) return st;
    int dev = params->device;
    if (dev < 0) {
        cudaError_t e = cudaGetDevice(&dev);
        if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
    } else {
        cudaError_t e = cudaSetDevice(dev);
        if (e != cudaSuccess) return cuda_fail(e, "cudaSetDevice");
    }
    dvm_plan_s *P = new (std::nothrow) dvm_plan_s();
    if (!P) {
        set_error("host allocation failed");
        return DVM_E_NOMEM;
    }
    P->d = params->d;
    P->N = params->N;
    P->p = 0;
    while ((1 << P->p) < P->N) ++P->p;
    P->Nbar = params->Nbar;
    P->Ntilde = Nt;
    P->kernel = params->kernel;
    P->device = dev;
    P->L = L;
    P->h = 2.0 * L / P->N;
    P->stream = (cudaStream_t)params->stream;
    P->shard_rank = params->shard_rank;
    P->shard_world = params->shard_world;
    P->pk.d = P->d;
    P->pk.p = P->p;
    P->pk.N = P->N;
    P->pk.H = 0;
    P->pk.mask = 0;
    for (int j = 0; j < P->d; ++j) {
        P->pk.H = (P->pk.H << P->p) | (1u << (P->p - 1));
        P->pk.mask = (P->pk.mask << P->p) | (uint32_t)(P->N - 1);
    }
    st = build_table(P);
    if (st) {
        free_table(P);
        delete P;
        return st;
    }
    *out = P;
    return DVM_OK;
}

dvm_status_t dvm_plan(int d, int N, int Nbar, dvm_kernel_t kernel, dvm_plan_t *out)
{
    dvm_plan_params_t p;
    memset(&p, 0, sizeof(p));
    p.d = d;
    p.N = N;
    p.Nbar = Nbar;
    p.Ntilde = 0;
    p.L = 8.0;
    p.kernel = kernel;
    p.device = -1;
    p.stream = nullptr;
    p.shard_rank = 0;
    p.shard_world = 1;
    return dvm_plan_ex(&p, out);
}

dvm_status_t dvm_plan_info(dvm_plan_t P, dvm_plan_info_t *info)
{
    if (!P || !info) {
        set_error("NULL argument");
        return DVM_E_NULL;
    }
    info->d = P->d;
    info->N = P->N;
    info->Nbar = P->Nbar;
    info->Ntilde = P->Ntilde;
    info->kernel = P->kernel;
    info->A = P->A;
    info->A_local = (int)P->local.size();
    info->rows_total = P->R;
    info->nodes = nodes_of(P);
    info->L = P->L;
    info->h = P->h;
    const Workspace &w = P->ws;
    // every device buffer the plan holds: tables, evaluation workspaces, staging
    const int64_t nd = nodes_of(P);
    size_t bytes = P->table_bytes + P->g.bytes;
    bytes += sizeof(double) * (size_t)w.slots * w.slot_elems * ((w.S ? 1 : 0) + (w.part ? 1 : 0));
    bytes += sizeof(double) * 2 * w.stage_elems;
    bytes += sizeof(double2) * (w.fft_z_elems + w.g3_f_elems + w.g3_t_elems + w.g3_q_elems + w.sp_z_elems +
                                w.fg_fhat_elems);
    bytes += sizeof(unsigned int) * w.g3_ctr_elems;
    bytes += sizeof(double) * (w.p2_scr_elems + w.p2_part_elems);
    bytes += sizeof(double) * (size_t)nd * ((w.qtmp ? 1 : 0) + (w.f1tmp ? 1 : 0));
    bytes += sizeof(double) * (kMaxD + 2) * w.mom_rows;
    bytes += sizeof(double2) * w.f32_z_elems + sizeof(double) * w.f32_part_elems;
    bytes += sizeof(double) * (w.lv_f_elems + w.lv_q_elems) + sizeof(int64_t) * w.lv_idx_elems +
             sizeof(int) * w.lv_cnt_elems;
    info->workspace_bytes = bytes;
    info->launches = P->launches;
    return DVM_OK;
}

dvm_status_t dvm_plan_directions(dvm_plan_t P, int *dirs, int *M, double *a, int *local)
{
    if (!P) {
        set_error("NULL argument");
        return DVM_E_NULL;
    }
    for (int i = 0; i < P->A; ++i) {
        if (dirs)
            for (int j = 0; j < P->d; ++j) dirs[i * P->d + j] = P->h_e[3 * i + j];
        if (M) M[i] = P->h_M[i];
        if (a) a[i] = P->h_a[i];
        if (local) local[i] = P->is_local[i];
    }
    return DVM_OK;
}

dvm_status_t dvm_plan_geometry(dvm_plan_t P, int idx, int *u, int *w, int *nrows, int *b, int *lo, int *hi,
                               int cap)
{
    if (!P || !nrows) {
        set_error("NULL argument");
        return DVM_E_NULL;
    }
    if (idx < 0 || idx >= P->A) {
        set_error("direction index out of range");
        return DVM_E_SHAPE;
    }
    int uu[3], ww[3];
    DVM_CUDA(cudaMemcpyAsync(uu, P->t.u + 3 * idx, sizeof(uu), cudaMemcpyDeviceToHost, P->stream));
    DVM_CUDA(cudaMemcpyAsync(ww, P->t.w + 3 * idx, sizeof(ww), cudaMemcpyDeviceToHost, P->stream));
    const int r0 = P->h_row_off[idx], n = P->h_row_off[idx + 1] - r0;
    const int m = n < cap ? n : cap;
    if (m > 0 && b) DVM_CUDA(cudaMemcpyAsync(b, P->t.row_b + r0, sizeof(int) * m, cudaMemcpyDeviceToHost, P->stream));
    if (m > 0 && lo) DVM_CUDA(cudaMemcpyAsync(lo, P->t.row_lo + r0, sizeof(int) * m, cudaMemcpyDeviceToHost, P->stream));
    if (m > 0 && hi) DVM_CUDA(cudaMemcpyAsync(hi, P->t.row_hi + r0, sizeof(int) * m, cudaMemcpyDeviceToHost, P->stream));
    DVM_CUDA(cudaStreamSynchronize(P->stream));
    for (int j = 0; j < P->d; ++j) {
        if (u) u[j] = uu[j];
        if (w) w[j] = ww[j];
    }
    *nrows = n;
    return DVM_OK;
}

dvm_status_t dvm_set_stream(dvm_plan_t P, void *stream)
{
    if (!P) {
        set_error("NULL argument");
        return DVM_E_NULL;
    }
    P->stream = (cudaStream_t)stream;
    return DVM_OK;
}

dvm_status_t dvm_collide_batched(dvm_plan_t P, const double *f, double *Q, int64_t ncells, int64_t cell_stride)
{
    NvtxRange nvtx_range("dvm_collide_batched");
    dvm_status_t st = check_batch(P, f, Q, ncells, &cell_stride);
    if (st) return st;
    return run_cached(P, 0, f, Q, ncells, cell_stride,
                      [&]() { return collide_batched(P, f, Q, ncells, cell_stride); });
}

dvm_status_t dvm_collide_batched_levels(const dvm_plan_t *plans, int nlevels, const double *f, double *Q,
                                        int64_t ncells, int64_t cell_stride, const int *level)
{
    NvtxRange nvtx_range("dvm_collide_batched_levels");
    if (!plans || nlevels < 1 || (ncells > 0 && !level)) {
        set_error(nlevels < 1 ? "nlevels must be >= 1" : "NULL argument");
        return nlevels < 1 ? DVM_E_SHAPE : DVM_E_NULL;
    }
    if (nlevels > 64) {
        set_error("at most 64 levels");
        return DVM_E_SHAPE;
    }
    for (int i = 0; i < nlevels; ++i) {
        const dvm_plan_s *a = plans[0], *b = plans[i];
        if (!b) {
            set_error("NULL plan");
            return DVM_E_NULL;
        }
        if (b->d != a->d || b->N != a->N || b->Ntilde != a->Ntilde || b->L != a->L || b->kernel != a->kernel ||
            b->device != a->device || b->stream != a->stream || b->shard_world != a->shard_world ||
            b->shard_rank != a->shard_rank) {
            set_error("dvm_collide_batched_levels: the plans must share d, N, Ñ, L, kernel, device, stream and "
                      "shard (they may differ only in N̄)");
            return DVM_E_STATE;
        }
    }
    dvm_status_t st = check_batch(plans[0], f, Q, ncells, &cell_stride);
    if (st) return st;
    return collide_levels(plans, nlevels, f, Q, ncells, cell_stride, level);
}

dvm_status_t dvm_collide_push(dvm_plan_t P, const double *f, int64_t ncells, void *const *windows, int rank,
                              int world, unsigned int epoch)
{
    NvtxRange nvtx_range("dvm_collide_push");
    double *mine = nullptr;
    dvm_status_t st = peer_push_check(P, f, ncells, windows, rank, world, epoch, &mine);
    if (st) return st;
    // the evaluation and the push of a repeated call replay one captured graph
    // (kind 2, keyed by f and the local slot); another window set invalidates it
    uint64_t key = 1469598103934665603ull;
    for (int r = 0; r < world; ++r) key = (key ^ (uint64_t)(uintptr_t)windows[r]) * 1099511628211ull;
    key = (key ^ (uint64_t)world) * 1099511628211ull;
    if (key != P->peer_key) {
        P->peer_key = key;
        ++P->version;
    }
    const int64_t nodes = nodes_of(P);
    return run_cached(P, 2, f, mine, ncells, nodes, [&]() -> dvm_status_t {
        dvm_status_t s2 = collide_batched(P, f, mine, ncells, nodes);
        if (s2) return s2;
        return peer_push_launch(P, mine, ncells * nodes, windows, rank, world);
    });
}

dvm_status_t dvm_collide(dvm_plan_t P, const double *f, double *Q)
{
    return dvm_collide_batched(P, f, Q, 1, 0);
}

dvm_status_t dvm_collide_batched_host(dvm_plan_t P, const double *f_host, double *Q_host, int64_t ncells,
                                      int64_t cell_stride)
{
    NvtxRange nvtx_range("dvm_collide_batched_host");
    dvm_status_t st = check_batch(P, f_host, Q_host, ncells, &cell_stride);
    if (st) return st;
    if (ncells == 0) return DVM_OK;
    const int64_t nodes = nodes_of(P);
    const size_t elems = (size_t)ncells * nodes;
    Workspace &w = P->ws;
    if (w.stage_elems < elems) {
        DVM_CUDA(cudaStreamSynchronize(P->stream));
        if (w.f_stage) cudaFree(w.f_stage);
        if (w.q_stage) cudaFree(w.q_stage);
        w.f_stage = w.q_stage = nullptr;
        w.stage_elems = 0;
        if (cudaMalloc(&w.f_stage, sizeof(double) * elems) != cudaSuccess ||
            cudaMalloc(&w.q_stage, sizeof(double) * elems) != cudaSuccess) {
            if (w.f_stage) cudaFree(w.f_stage);
            w.f_stage = w.q_stage = nullptr;
            set_error("staging allocation failed");
            return DVM_E_NOMEM;
        }
        w.stage_elems = elems;
    }
    // Large batches are pipelined in 4 chunks of whole cell pairs: the host->device
    // copy of chunk i + 1 and the device->host copy of chunk i - 1 run on two
    // plan-owned copy streams while chunk i is evaluated on the plan's stream
    // (pinned host buffers needed for the overlap; results equal a one-shot call
    // up to the FFT loss's cell pairing, which chunks of even size preserve).
    const int nch = ncells >= 256 ? 4 : 1;
    const int64_t per = nch == 1 ? ncells : (((ncells + nch - 1) / nch) + 1) / 2 * 2;
    auto copy = [&](double *dst, int64_t dpitch, const double *src, int64_t spitch, int64_t nc, cudaMemcpyKind k,
                    cudaStream_t strm) -> cudaError_t {
        if (dpitch == nodes && spitch == nodes)
            return cudaMemcpyAsync(dst, src, sizeof(double) * (size_t)(nc * nodes), k, strm);
        return cudaMemcpy2DAsync(dst, sizeof(double) * dpitch, src, sizeof(double) * spitch, sizeof(double) * nodes,
                                 nc, k, strm);
    };
    if (nch == 1) {
        // small batches: copy in, evaluate, copy out, all on the plan's stream
        // (no copy streams or events: their cross-stream waits cost more than
        // the overlap they could buy)
        cudaError_t ce0 = copy(w.f_stage, nodes, f_host, cell_stride, ncells, cudaMemcpyHostToDevice, P->stream);
        if (ce0 != cudaSuccess) return cuda_fail(ce0, "host->device copy");
        st = run_cached(P, 0, w.f_stage, w.q_stage, ncells, nodes,
                        [&]() { return collide_batched(P, w.f_stage, w.q_stage, ncells, nodes); });
        if (st) return st;
        ce0 = copy(Q_host, cell_stride, w.q_stage, nodes, ncells, cudaMemcpyDeviceToHost, P->stream);
        if (ce0 != cudaSuccess) return cuda_fail(ce0, "device->host copy");
        const cudaError_t ce = cudaStreamSynchronize(P->stream);
        if (ce != cudaSuccess) return cuda_fail(ce, "cudaStreamSynchronize");
        return DVM_OK;
    }
    if (!P->cstream[0]) {
        DVM_CUDA(cudaStreamCreateWithFlags(&P->cstream[0], cudaStreamNonBlocking));
        DVM_CUDA(cudaStreamCreateWithFlags(&P->cstream[1], cudaStreamNonBlocking));
    }
    std::vector<cudaEvent_t> ev;
    auto fail = [&](dvm_status_t code) {
        for (cudaEvent_t e : ev) cudaEventDestroy(e);
        return code;
    };
    for (int i = 0; i < 3 * nch; ++i) {
        cudaEvent_t e;
        if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) return fail(cuda_fail(cudaGetLastError(), "cudaEventCreate"));
        ev.push_back(e);
    }
    // ev[0]: previous work on the plan's stream is done with the staging buffers
    cudaError_t ce = cudaEventRecord(ev[0], P->stream);
    if (ce == cudaSuccess) ce = cudaStreamWaitEvent(P->cstream[0], ev[0], 0);
    if (ce != cudaSuccess) return fail(cuda_fail(ce, "cudaStreamWaitEvent"));
    for (int i = 0; i < nch; ++i) {  // all host->device copies, in order, on copy stream 0
        const int64_t c0 = i * per, nc = std::min<int64_t>(per, ncells - c0);
        if (nc <= 0) break;
        ce = copy(w.f_stage + c0 * nodes, nodes, f_host + c0 * cell_stride, cell_stride, nc, cudaMemcpyHostToDevice,
                  P->cstream[0]);
        if (ce == cudaSuccess) ce = cudaEventRecord(ev[nch + i], P->cstream[0]);
        if (ce != cudaSuccess) return fail(cuda_fail(ce, "host->device copy"));
    }
    for (int i = 0; i < nch; ++i) {
        const int64_t c0 = i * per, nc = std::min<int64_t>(per, ncells - c0);
        if (nc <= 0) break;
        if ((ce = cudaStreamWaitEvent(P->stream, ev[nch + i], 0)) != cudaSuccess) return fail(cuda_fail(ce, "wait"));
        if ((st = collide_batched(P, w.f_stage + c0 * nodes, w.q_stage + c0 * nodes, nc, nodes))) return fail(st);
        ce = cudaEventRecord(ev[2 * nch + i], P->stream);
        if (ce == cudaSuccess) ce = cudaStreamWaitEvent(P->cstream[1], ev[2 * nch + i], 0);
        if (ce == cudaSuccess)
            ce = copy(Q_host + c0 * cell_stride, cell_stride, w.q_stage + c0 * nodes, nodes, nc, cudaMemcpyDeviceToHost,
                      P->cstream[1]);
        if (ce != cudaSuccess) return fail(cuda_fail(ce, "device->host copy"));
    }
    ce = cudaStreamSynchronize(P->cstream[1]);
    if (ce == cudaSuccess) ce = cudaStreamSynchronize(P->stream);
    for (cudaEvent_t e : ev) cudaEventDestroy(e);
    if (ce != cudaSuccess) return cuda_fail(ce, "cudaStreamSynchronize");
    return DVM_OK;
}

dvm_status_t dvm_moments(dvm_plan_t P, const double *f, double *out_host)
{
    if (!P || !f || !out_host) {
        set_error("NULL argument");
        return DVM_E_NULL;
    }
    Workspace &w = P->ws;
    if (!w.mom_dev || w.mom_rows < 1) {
        if (w.mom_dev) cudaFree(w.mom_dev);
        DVM_CUDA(cudaMalloc(&w.mom_dev, sizeof(double) * (kMaxD + 2)));
        w.mom_rows = 1;
    }
    dvm_status_t st = moments(P, f, w.mom_dev);
    if (st) return st;
    double tmp[kMaxD + 2];
    DVM_CUDA(cudaMemcpyAsync(tmp, w.mom_dev, sizeof(double) * (kMaxD + 2), cudaMemcpyDeviceToHost, P->stream));
    DVM_CUDA(cudaStreamSynchronize(P->stream));
    for (int k = 0; k < P->d + 2; ++k) out_host[k] = tmp[k];
    return DVM_OK;
}

// One explicit step of `scheme` (1: Euler f += dt Q(f); 2: TVD-RK2 / Heun,
// f1 = f + dt Q(f), f = (f + f1 + dt Q(f1)) / 2), then the
// moments row (device counter) if requested.
static dvm_status_t one_step(dvm_plan_s *P, int scheme, double *f, double dt, bool mom)
{
    const int64_t nodes = nodes_of(P);
    Workspace &w = P->ws;
    dvm_status_t st;
    // small 2D grids, Euler: unit sum, f += dt Q and the moments partials in one launch
    if (scheme == 1 && !P->wt.on && (P->path_mode == 0 || P->path_mode == 5) && w.mom_partial) {
        bool handled = false;
        int nb = 0;
        if ((st = euler_small2d(P, f, w.qtmp, dt, w.mom_partial, &nb, &handled))) return st;
        if (handled) {
            if (mom && (st = moments_final_ctr(P, nb, w.mom_dev, w.mom_ctr))) return st;
            return DVM_OK;
        }
    }
    if ((st = collide_batched(P, f, w.qtmp, 1, nodes))) return st;
    if (scheme == 1) {
        if ((st = axpy(P, f, w.qtmp, dt))) return st;
    } else {
        if ((st = rk2_stage(P, 1, f, w.f1tmp, w.qtmp, dt))) return st;
        if ((st = collide_batched(P, w.f1tmp, w.qtmp, 1, nodes))) return st;
        if ((st = rk2_stage(P, 2, f, w.f1tmp, w.qtmp, dt))) return st;
    }
    if (mom && (st = moments_ctr(P, f, w.mom_dev, w.mom_ctr))) return st;
    return DVM_OK;
}

// nsteps steps of `scheme`; step 1 runs directly (it sizes every workspace),
// steps 2..nsteps replay one captured CUDA graph of a step on a plan-owned
// stream joined to the plan's stream by events (the launch-bound loop of the
// small grids).  Moments rows: 0 = initial state, s = after step s.
static dvm_status_t time_stepper(dvm_plan_s *P, int scheme, double *f, double dt, int nsteps, double *moments_host)
{
    if (!P || !f) {
        set_error("NULL argument");
        return DVM_E_NULL;
    }
    if (nsteps < 0 || !isfinite(dt)) {
        set_error("bad nsteps / dt");
        return DVM_E_SHAPE;
    }
    const int64_t nodes = nodes_of(P);
    Workspace &w = P->ws;
    const size_t rows = (size_t)nsteps + 1;
    const bool mom = moments_host != nullptr;
    if (!w.mom_dev || w.mom_rows < rows) {
        DVM_CUDA(cudaStreamSynchronize(P->stream));
        if (w.mom_dev) cudaFree(w.mom_dev);
        w.mom_dev = nullptr;
        DVM_CUDA(cudaMalloc(&w.mom_dev, sizeof(double) * (kMaxD + 2) * rows));
        w.mom_rows = rows;
    }
    if (!w.qtmp) DVM_CUDA(cudaMalloc(&w.qtmp, sizeof(double) * nodes));
    if (scheme == 2 && !w.f1tmp) DVM_CUDA(cudaMalloc(&w.f1tmp, sizeof(double) * nodes));
    if (!w.mom_ctr) DVM_CUDA(cudaMalloc(&w.mom_ctr, sizeof(int)));
    if (!w.mom_partial) DVM_CUDA(cudaMalloc(&w.mom_partial, sizeof(double) * 128 * (kMaxD + 2)));
    DVM_CUDA(cudaMemsetAsync(w.mom_ctr, 0, sizeof(int), P->stream));
    dvm_status_t st;
    if (mom && (st = moments_ctr(P, f, w.mom_dev, w.mom_ctr))) return st;
    if (nsteps >= 1 && (st = one_step(P, scheme, f, dt, mom))) return st;
    int done = nsteps >= 1 ? 1 : 0;
    if (nsteps >= 2 && P->use_graphs) {
        if (!P->gstream) {
            DVM_CUDA(cudaStreamCreateWithFlags(&P->gstream, cudaStreamNonBlocking));
            DVM_CUDA(cudaEventCreateWithFlags(&P->gev[0], cudaEventDisableTiming));
            DVM_CUDA(cudaEventCreateWithFlags(&P->gev[1], cudaEventDisableTiming));
        }
        DVM_CUDA(cudaEventRecord(P->gev[0], P->stream));
        DVM_CUDA(cudaStreamWaitEvent(P->gstream, P->gev[0], 0));
        cudaStream_t user = P->stream;
        const bool prof = P->profiling;
        const uint64_t l0 = P->launches;
        P->stream = P->gstream;
        P->profiling = false;  // no event records inside the captured step
        cudaGraph_t graph = nullptr;
        cudaGraphExec_t exec = nullptr;
        cudaError_t ce = cudaStreamBeginCapture(P->gstream, cudaStreamCaptureModeThreadLocal);
        if (ce == cudaSuccess) {
            st = one_step(P, scheme, f, dt, mom);
            ce = cudaStreamEndCapture(P->gstream, &graph);
            if (st == DVM_OK && ce == cudaSuccess) ce = cudaGraphInstantiate(&exec, graph, 0);
        }
        const uint64_t per_step = P->launches - l0;
        P->stream = user;
        P->profiling = prof;
        if (st == DVM_OK && ce == cudaSuccess && exec) {
            for (int s = done; s < nsteps; ++s) {
                ce = cudaGraphLaunch(exec, P->gstream);
                if (ce != cudaSuccess) break;
            }
            P->launches += per_step * (uint64_t)(nsteps - done - 1);  // the capture counted one step
            if (ce == cudaSuccess) done = nsteps;
        } else {
            P->launches = l0;
            cudaGetLastError();  // capture unsupported here: fall back to direct launches
            st = DVM_OK;
        }
        if (exec) cudaGraphExecDestroy(exec);
        if (graph) cudaGraphDestroy(graph);
        DVM_CUDA(cudaEventRecord(P->gev[1], P->gstream));
        DVM_CUDA(cudaStreamWaitEvent(P->stream, P->gev[1], 0));
        if (ce != cudaSuccess && done != nsteps) return cuda_fail(ce, "cudaGraphLaunch");
    }
    for (int s = done; s < nsteps; ++s)
        if ((st = one_step(P, scheme, f, dt, mom))) return st;
    if (mom) {
        std::string buf;
        buf.resize(sizeof(double) * (kMaxD + 2) * rows);
        DVM_CUDA(cudaMemcpyAsync(&buf[0], w.mom_dev, buf.size(), cudaMemcpyDeviceToHost, P->stream));
        DVM_CUDA(cudaStreamSynchronize(P->stream));
        const double *src = (const double *)buf.data();
        for (size_t r = 0; r < rows; ++r)
            for (int k = 0; k < P->d + 2; ++k) moments_host[r * (P->d + 2) + k] = src[r * (kMaxD + 2) + k];
    } else {
        DVM_CUDA(cudaStreamSynchronize(P->stream));
    }
    return DVM_OK;
}

dvm_status_t dvm_copy_cells(dvm_plan_t P, const double *src, const int64_t *src_idx, double *dst,
                            const int64_t *dst_idx, int64_t ncells)
{
    if (!P || !src || !dst) {
        set_error("NULL argument");
        return DVM_E_NULL;
    }
    if (ncells < 0) {
        set_error("ncells < 0");
        return DVM_E_SHAPE;
    }
    return copy_cells(P, src, src_idx, dst, dst_idx, ncells);
}

dvm_status_t dvm_euler(dvm_plan_t P, double *f, double dt, int nsteps, double *moments_host)
{
    NvtxRange nvtx_range("dvm_euler");
    return time_stepper(P, 1, f, dt, nsteps, moments_host);
}

dvm_status_t dvm_rk2(dvm_plan_t P, double *f, double dt, int nsteps, double *moments_host)
{
    NvtxRange nvtx_range("dvm_rk2");
    return time_stepper(P, 2, f, dt, nsteps, moments_host);
}

dvm_status_t dvm_set_graphs(dvm_plan_t P, int enable)
{
    if (!P) {
        set_error("NULL argument");
        return DVM_E_NULL;
    }
    ++P->version;  // invalidates a captured collide graph
    P->use_graphs = enable != 0;
    return DVM_OK;
}

dvm_status_t dvm_profile_enable(dvm_plan_t P, int enable)
{
    if (!P) {
        set_error("NULL argument");
        return DVM_E_NULL;
    }
    DVM_CUDA(cudaStreamSynchronize(P->stream));
    clear_profile(P);
    P->profiling = enable != 0;
    return DVM_OK;
}

static const char *kClassNames[] = {"k_linesum", "k_rowsum", "k_reduce", "k_zero", "k_moments", "k_axpy", "plan",
                                    "k_gain3d", "k_fft", "k_fg2", "k_small2d", "k_wline2d", "k_pair2d", "k_fg32"};

const char *dvm_profile_name(int k) { return (k >= 0 && k < KC_COUNT) ? kClassNames[k] : nullptr; }

dvm_status_t dvm_profile_read(dvm_plan_t P, double *ms, uint64_t *count, int n)
{
    if (!P || !ms || !count) {
        set_error("NULL argument");
        return DVM_E_NULL;
    }
    DVM_CUDA(cudaStreamSynchronize(P->stream));
    for (int k = 0; k < n; ++k) {
        ms[k] = 0.0;
        count[k] = 0;
    }
    for (auto &r : P->prof) {
        if (r.cls >= n) continue;
        float t = 0.f;
        DVM_CUDA(cudaEventElapsedTime(&t, r.a, r.b));
        ms[r.cls] += t;
        count[r.cls] += 1;
    }
    return DVM_OK;
}

dvm_status_t dvm_set_path(dvm_plan_t P, int path)
{
    if (!P) {
        set_error("NULL argument");
        return DVM_E_NULL;
    }
    ++P->version;  // invalidates a captured collide graph
    if (path < 0 || path > 7) {
        set_error("path must be 0 (auto), 1 (v1 orbit sweeps), 2 (gain3d / pair2d line walks), 3 (spectral "
                  "reference), 4 (3D FFT gain), 5 (2D small grids), 6 (3D N = 32 spectral direction pairs) or 7 "
                  "(2D tiles)");
        return DVM_E_STATE;
    }
    P->path_mode = path;
    return DVM_OK;
}

dvm_status_t dvm_set_tuning(dvm_plan_t P, const char *key, int value)
{
    if (!P || !key) {
        set_error("NULL argument");
        return DVM_E_NULL;
    }
    ++P->version;  // invalidates a captured collide graph
    const std::string k(key);
    auto bad = [&]() {
        set_error("dvm_set_tuning: bad value for " + k);
        return DVM_E_STATE;
    };
    if (k == "max_groups") {
        if (value < 0) return bad();
        P->tune.max_groups = value;
    } else if (k == "ring_slots") {
        if (value != 0 && (value < 2 || value > 4)) return bad();
        P->tune.ring_slots = value;
    } else if (k == "fg_chunks") {
        if (value < 0 || value > 64) return bad();
        P->tune.fg_chunks = value;
    } else if (k == "g3_cl") {
        if (value != 0 && value != 4 && value != 8 && value != 16) return bad();
        P->tune.g3_cl = value;
    } else if (k == "verbose") {
        P->tune.verbose = value != 0;
    } else if (k == "timing_dbg") {
        if (value < 0 || value > 7) return bad();
        P->tune.fg_dbg = value;
    } else {
        set_error("dvm_set_tuning: unknown key " + k);
        return DVM_E_STATE;
    }
    return DVM_OK;
}

dvm_status_t dvm_set_weights(dvm_plan_t P, const double *a_box, const double *b_box)
{
    if (!P) {
        set_error("NULL argument");
        return DVM_E_NULL;
    }
    ++P->version;  // invalidates a captured collide graph
    return set_weights(P, a_box, b_box);
}

dvm_status_t dvm_sync(dvm_plan_t P)
{
    if (!P) {
        set_error("NULL argument");
        return DVM_E_NULL;
    }
    DVM_CUDA(cudaStreamSynchronize(P->stream));
    DVM_CUDA(cudaGetLastError());
    return DVM_OK;
}

dvm_status_t dvm_plan_destroy(dvm_plan_t P)
{
    if (!P) {
        set_error("NULL argument");
        return DVM_E_NULL;
    }
    cudaStreamSynchronize(P->stream);
    if (P->cg.exec) cudaGraphExecDestroy(P->cg.exec);
    if (P->gstream) {
        cudaStreamSynchronize(P->gstream);
        cudaStreamDestroy(P->gstream);
        cudaEventDestroy(P->gev[0]);
        cudaEventDestroy(P->gev[1]);
    }
    for (cudaStream_t &cs : P->cstream)
        if (cs) {
            cudaStreamSynchronize(cs);
            cudaStreamDestroy(cs);
            cs = nullptr;
        }
    free_workspace(P);
    free_table(P);
    delete P;
    return DVM_OK;
}

}  // extern "C"
