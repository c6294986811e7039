// The C-ABI runtime (include/swb.h): device memory, streams, the time loop, halo linking.
// It replaces the reference Engine (src/executor.cpp:140-606) for the acoustic IET.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <map>
#include <mutex>
#include <cmath>
#include <cstdio>
#include <climits>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/swb.h"
#include "kernels.h"
#include "swb_internal.h"

using namespace swb;

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
    g_err = msg;
    return code;
}

#define SWB_CUDA(call)                                                                     \
    do {                                                                                   \
        cudaError_t e_ = (call);                                                           \
        if (e_ != cudaSuccess)                                                             \
            return fail(SWB_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e_));    \
    } while (0)

constexpr uint32_t kBlobMagic = 0x53574231u;  // "SWB1"

// Process-wide cache of the large per-handle buffers (u levels, m, damp), keyed by device and
// exact size: a handle created after another one was destroyed (a new problem of the same
// grid, the bench's end-to-end run) reuses its HBM instead of paying cudaMalloc/cudaFree
// (milliseconds each for hundreds of MB).  SWB_NO_POOL=1 disables it.
struct BufPool {
    std::mutex mu;
    std::multimap<std::pair<int, size_t>, void*> free_;
};
BufPool& pool() {
    static BufPool* p = new BufPool();  // never destroyed: outlives static handles at exit
    return *p;
}
bool pool_enabled() {
    static const bool on = std::getenv("SWB_NO_POOL") == nullptr;
    return on;
}
cudaError_t pool_alloc(int device, void** ptr, size_t bytes) {
    if (pool_enabled()) {
        std::lock_guard<std::mutex> lk(pool().mu);
        auto it = pool().free_.find({device, bytes});
        if (it != pool().free_.end()) {
            *ptr = it->second;
            pool().free_.erase(it);
            return cudaSuccess;
        }
    }
    cudaError_t e = cudaMalloc(ptr, bytes);
    if (e == cudaErrorMemoryAllocation && pool_enabled()) {  // give the cache back and retry
        cudaGetLastError();
        std::lock_guard<std::mutex> lk(pool().mu);
        for (auto it = pool().free_.begin(); it != pool().free_.end();) {
            if (it->first.first == device) {
                cudaFree(it->second);
                it = pool().free_.erase(it);
            } else {
                ++it;
            }
        }
        e = cudaMalloc(ptr, bytes);
    }
    return e;
}
void pool_free(int device, void* ptr, size_t bytes, bool shared = false) {
    if (!ptr) return;
    if (!pool_enabled() || shared) {  // IPC-exported memory may still be mapped by a peer
        cudaFree(ptr);
        return;
    }
    std::lock_guard<std::mutex> lk(pool().mu);
    pool().free_.insert({{device, bytes}, ptr});
}

struct IpcBlob {
    uint32_t magic;
    int32_t xg_off, nl0, n1, n2, P2, H;
    int32_t fused_capable, grid;
    int64_t level_floats;
    cudaIpcMemHandle_t u_handle;
    cudaIpcMemHandle_t flag_handle;
    unsigned char uuid[16];  // device of the exporting handle
};

// Fused in-kernel halo ordering needs both slabs' persistent grids resident at once: true on two
// devices, not when two processes share one GPU (then the wait/signal kernels order the steps).
bool same_device(int device, const unsigned char* uuid) {
    cudaDeviceProp prop{};
    if (cudaGetDeviceProperties(&prop, device) != cudaSuccess) return false;
    return std::memcmp(prop.uuid.bytes, uuid, 16) == 0;
}

// Ordinal (in this process's enumeration) of the device with this UUID, or -2 if not visible.
int device_of_uuid(const unsigned char* uuid) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) return -2;
    for (int d = 0; d < n; ++d) {
        cudaDeviceProp prop{};
        if (cudaGetDeviceProperties(&prop, d) == cudaSuccess && std::memcmp(prop.uuid.bytes, uuid, 16) == 0) return d;
    }
    return -2;
}

}  // namespace

struct swb_handle {
    // small device buffers (sizes kept for the pool): see hbuf_alloc
    std::vector<std::pair<void*, size_t>> hbufs;
    int device = 0;
    cudaStream_t stream = nullptr;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    int n0 = 0, n1 = 0, n2 = 0, so = 0, H = 0, HU = 0, P2 = 0;
    int lo = 0, hi = 0, gb = 0, ga = 0, nl0 = 0, xg_off = 0;
    long long plane = 0, level_floats = 0;
    int form = 0;
    float* u = nullptr;
    float* m = nullptr;
    float* damp = nullptr;
    float* d_wavelet = nullptr;
    int wavelet_len = 0;
    unsigned* d_smax = nullptr;
    int smax_cap = 0;
    unsigned* d_ring = nullptr;  // [3]
    bool ring_dirty = true;
    // receivers
    int n_rec = 0;
    std::vector<int> rec_owned;          // global receiver index per owned receiver
    long long* d_rec_idx = nullptr;      // [owned][8] local flat corner indices (-1: not owned)
    double* d_rec_w = nullptr;           // [owned][8] corner weights
    float* d_traces = nullptr;
    int traces_cap = 0;
    // adjoint: per owned receiver corner, w_c / (m + damp dt/2) (0 outside the update interior),
    // and the source-point sampling stencil (index + dt^2 (m_s + g_s) / m_s)
    double* d_inj_w = nullptr;
    long long* d_src_idx = nullptr;
    double* d_src_w = nullptr;
    float* d_adj = nullptr;        // [nt][owned] receiver data of the running adjoint
    float* d_src_trace = nullptr;  // [nt]
    int adj_cap = 0;
    // snapshots (swb_apply_snapshots): device staging ring + two copy streams
    static constexpr int kSnapSlots = 2;
    float* d_stage[kSnapSlots] = {nullptr, nullptr};
    cudaStream_t s_d2d = nullptr, s_d2h = nullptr;
    cudaEvent_t ev_step = nullptr, ev_d2d[kSnapSlots] = {nullptr, nullptr}, ev_d2h[kSnapSlots] = {nullptr, nullptr};
    // stencil
    Geo geo{};
    Coef K{};
    Ctl ctl{};
    Peer peer{};
    TmaPlan plan{};
    alignas(128) unsigned char maps[kTmaMapsBytes];
    bool use_tma = false;
    unsigned char* d_dflag = nullptr;
    unsigned long long* d_trace = nullptr;  // SWB_TRACE: per-CTA timestamps of the last launch
    // halo links
    unsigned long long* d_flags = nullptr;   // [0]: written by lower neighbour, [1]: by upper
    unsigned* d_err = nullptr;                // halo-exchange timeout flag
    unsigned long long* lo_remote = nullptr; // lower neighbour's d_flags[1]
    unsigned long long* hi_remote = nullptr; // upper neighbour's d_flags[0]
    // per side: 1 = fused in-kernel ordering (both ends run the TMA kernel), 0 = wait/signal kernels
    int fused_lo = 0, fused_hi = 0;
    int nb_grid_lo = 0, nb_grid_hi = 0;      // neighbours' CTAs per step (fused counters)
    int peer_dev_lo = -1, peer_dev_hi = -1;  // neighbours' device ordinals (-2: another process's)
    void* ipc_lo_u = nullptr;
    void* ipc_hi_u = nullptr;
    void* ipc_lo_f = nullptr;
    void* ipc_hi_f = nullptr;
    unsigned long long steps_done = 0;
    bool exported = false;  // u was exported through CUDA IPC (never recycled through the pool)
    // pending apply
    int pend_step0 = 0, pend_nt = 0;
    bool pending = false;
    swb_stats stats{};
    uint64_t launches = 0;
};

namespace {

int setup_device(int device) {
    int count = 0;
    cudaError_t e = cudaGetDeviceCount(&count);
    if (e != cudaSuccess || count == 0)
        return fail(SWB_ECUDA, std::string("no CUDA device available (") +
                                   cudaGetErrorString(e) + "); there is no CPU fallback");
    if (device < 0 || device >= count) return fail(SWB_EINVAL, "device ordinal out of range");
    // architecture check once per device: two attribute queries (cudaGetDeviceProperties
    // costs milliseconds, which every handle creation would pay)
    static std::atomic<unsigned long long> checked{0};
    const unsigned long long bit = device < 64 ? (1ull << device) : 0ull;
    if (!(checked.load() & bit)) {
        int major = 0, minor = 0;
        SWB_CUDA(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device));
        SWB_CUDA(cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, device));
        if (major != 10) {
            cudaDeviceProp prop{};
            SWB_CUDA(cudaGetDeviceProperties(&prop, device));
            return fail(SWB_ECUDA, std::string("device ") + prop.name + " is sm_" +
                                       std::to_string(major * 10 + minor) +
                                       "; this library is built for sm_100a (B200) only");
        }
        checked.fetch_or(bit);
    }
    SWB_CUDA(cudaSetDevice(device));
    return SWB_OK;
}

// Small per-handle device buffers come from the same pool as the fields, so repeated handles
// of one problem (the bench's end-to-end runs, a solver re-creating operators) pay no
// cudaMalloc/cudaFree; the sizes are kept for pool_free in swb_destroy.
cudaError_t hbuf_alloc(swb_handle* h, void** ptr, size_t bytes) {
    cudaError_t e = pool_alloc(h->device, ptr, bytes);
    if (e == cudaSuccess) h->hbufs.emplace_back(*ptr, bytes);
    return e;
}
template <typename T>
cudaError_t hbuf_alloc(swb_handle* h, T** ptr, size_t bytes) {
    return hbuf_alloc(h, reinterpret_cast<void**>(ptr), bytes);
}
void hbuf_free(swb_handle* h, void* ptr) {
    if (!ptr) return;
    for (auto it = h->hbufs.begin(); it != h->hbufs.end(); ++it)
        if (it->first == ptr) {
            pool_free(h->device, ptr, it->second);
            h->hbufs.erase(it);
            return;
        }
    cudaFree(ptr);
}

void coef_from(const swb_problem* p, int H, const float* w, Coef& K) {
    std::memset(&K, 0, sizeof K);
    for (int k = 0; k <= H; ++k) K.c[k] = w[H + k];
    const double c0 = K.c[0], c1 = K.c[1];
    K.R_d = c0 + 2.0 * c1;
    K.R = static_cast<float>(K.R_d);
    for (int d = 0; d < 3; ++d) {
        K.h[d] = p->spacing[d];
        const double hd = static_cast<double>(p->spacing[d]);
        K.inv_h2[d] = 1.0 / (hd * hd);
    }
    K.dt = p->dt;
    const double dt = static_cast<double>(p->dt);
    K.inv_dt2 = 1.0 / (dt * dt);
    K.half_inv_dt = 0.5 / dt;
    K.inject = dt * dt;
    K.iso = (p->spacing[0] == p->spacing[1] && p->spacing[1] == p->spacing[2]) ? 1 : 0;
    K.R3 = static_cast<float>(3.0 * K.R_d);
    {
        double r = c0;
        for (int k = 1; k <= H; ++k) r += 2.0 * static_cast<double>(K.c[k]);
        K.R3f = static_cast<float>(3.0 * r);
        double rd = c0;
        for (int d = 0; d < 4; ++d) {
            if (d + 1 <= H) rd += 2.0 * static_cast<double>(K.c[d + 1]);
            K.R3k[d] = static_cast<float>(3.0 * rd);
        }
    }
    const double h0 = static_cast<double>(p->spacing[0]);
    const double kap = (dt / h0) * (dt / h0);
    K.kap_hi = static_cast<float>(kap);
    K.kap_lo = static_cast<float>(kap - static_cast<double>(K.kap_hi));
    K.half_dt = static_cast<float>(0.5 * dt);
}

int ensure_smax(swb_handle* h, int nt) {
    if (nt <= h->smax_cap) return SWB_OK;
    if (h->d_smax) SWB_CUDA(cudaStreamSynchronize(h->stream));
    hbuf_free(h, h->d_smax);
    h->d_smax = nullptr;
    int cap = std::max(nt, 1024);
    SWB_CUDA(hbuf_alloc(h, &h->d_smax, sizeof(unsigned) * cap));
    h->smax_cap = cap;
    return SWB_OK;
}

int ensure_traces(swb_handle* h, int nt) {
    const int owned = static_cast<int>(h->rec_owned.size());
    if (owned == 0) return SWB_OK;
    long long need = static_cast<long long>(nt) * owned;
    if (need <= h->traces_cap) return SWB_OK;
    if (h->d_traces) SWB_CUDA(cudaStreamSynchronize(h->stream));
    hbuf_free(h, h->d_traces);
    h->d_traces = nullptr;
    SWB_CUDA(hbuf_alloc(h, &h->d_traces, sizeof(float) * need));
    h->traces_cap = static_cast<int>(need);
    return SWB_OK;
}

int refresh_ring(swb_handle* h) {
    if (!h->ring_dirty) return SWB_OK;
    SWB_CUDA(cudaMemsetAsync(h->d_ring, 0, 3 * sizeof(unsigned), h->stream));
    // owned planes [gb, gb + hi - lo); interior = updated region
    const int own0 = h->gb, own1 = h->gb + (h->hi - h->lo);
    for (int l = 0; l < 3; ++l) {
        SWB_CUDA(launch_ring_max(h->u + l * h->level_floats, h->plane, h->P2, own0, own1, h->n1,
                                 h->n2, h->geo.x0, h->geo.x1, h->geo.y0, h->geo.y1, h->geo.z0,
                                 h->geo.z1, h->d_ring + l, h->stream));
    }
    h->ring_dirty = false;
    return SWB_OK;
}

bool linked(const swb_handle* h) { return h->lo_remote || h->hi_remote || h->peer.lo_lev[0] || h->peer.hi_lev[0]; }


int enqueue_steps(swb_handle* h, int step0, int nt, int slot0 = 0) {
    const int kmask = (h->lo_remote && !h->fused_lo ? 1 : 0) | (h->hi_remote && !h->fused_hi ? 2 : 0);
    int rec_pending = 0;  // steps since the last receiver sampling launch
    for (int i = 0; i < nt;) {
        const int s = step0 + i;
        if (kmask) {  // kernel-based ordering for sides without fused support
            SWB_CUDA(launch_wait_flags(h->d_flags, kmask, h->steps_done + i, h->d_err, h->stream));
            ++h->launches;
        }
        Ctl c = h->ctl;
        c.step = s;
        c.slot = slot0 + i;
        if (c.trace) c.trace += static_cast<size_t>(s & 1) * 8 * 1024;  // SWB_TRACE: even / odd step
        c.err = h->d_err;
        c.ghost_lo_end = 0;
        c.ghost_hi_begin = INT_MAX;
        if ((h->lo_remote && h->fused_lo) || (h->hi_remote && h->fused_hi)) {
            c.flags = h->d_flags;
            if (h->lo_remote && h->fused_lo) {
                c.sig_lo = h->lo_remote;
                c.need_lo = static_cast<unsigned long long>(h->nb_grid_lo) * (h->steps_done + i);
                c.ghost_lo_end = h->gb;
            }
            if (h->hi_remote && h->fused_hi) {
                c.sig_hi = h->hi_remote;
                c.need_hi = static_cast<unsigned long long>(h->nb_grid_hi) * (h->steps_done + i);
                c.ghost_hi_begin = h->gb + (h->hi - h->lo);
            }
        }
        if (h->use_tma) {
            SWB_CUDA(launch_tma(h->plan, h->maps, h->geo, h->K, c, h->peer, h->stream));
        } else {
            const int form = h->form == SWB_FORM_PLAIN_F64   ? 1
                             : h->form == SWB_FORM_PLAIN_F32 ? 2
                             : h->form == SWB_FORM_FACTORISED_SIMPLE_F32C ? 3
                                                                     : 0;
            SWB_CUDA(launch_simple(h->H, form, h->geo, h->K, c, h->peer, h->stream));
        }
        ++h->launches;
        if (!h->rec_owned.empty() && (++rec_pending == 3 || i == nt - 1)) {
            // receiver samples of the last rec_pending steps (step s' left its output in level
            // (s' + 1) % 3, which steps s' + 1 and s' + 2 do not write): one launch per three steps
            const int owned = static_cast<int>(h->rec_owned.size());
            const int j0 = i + 1 - rec_pending;
            const float* lev[3];
            for (int b = 0; b < rec_pending; ++b)
                lev[b] = h->u + ((step0 + j0 + b + 1) % 3) * h->level_floats;
            SWB_CUDA(launch_samplers_batch(lev, rec_pending, h->d_rec_idx, h->d_rec_w, owned,
                                           h->d_traces + static_cast<long long>(slot0 + j0) * owned, h->stream));
            ++h->launches;
            rec_pending = 0;
        }
        if (kmask) {
            SWB_CUDA(launch_signal_flags(kmask & 1 ? h->lo_remote : nullptr, kmask & 2 ? h->hi_remote : nullptr,
                                         h->steps_done + i + 1, h->stream));
            ++h->launches;
        }
        ++i;
    }
    h->steps_done += nt;
    return SWB_OK;
}

bool fused_capable(const swb_handle* h) { return h->use_tma; }

void compute_peer_ranges(swb_handle* h) {
    // planes mirrored to the lower neighbour: global [lo, lo+HU) ∩ updated; upper: [hi-HU, hi) ∩ updated
    Peer& p = h->peer;
    const int upd0 = h->geo.x0, upd1 = h->geo.x1;  // local
    if (p.lo_lev[0]) {
        p.lo_first = std::max(upd0, h->gb);
        p.lo_last = std::min(upd1, h->gb + h->HU);
    } else {
        p.lo_first = p.lo_last = 0;
    }
    if (p.hi_lev[0]) {
        const int own1 = h->gb + (h->hi - h->lo);
        p.hi_first = std::max(upd0, own1 - h->HU);
        p.hi_last = std::min(upd1, own1);
    } else {
        p.hi_first = p.hi_last = 0;
    }
    if (p.lo_first >= p.lo_last) p.lo_first = p.lo_last = 0;
    if (p.hi_first >= p.hi_last) p.hi_first = p.hi_last = 0;
}

}  // namespace

extern "C" {

const char* swb_last_error(void) { return g_err.c_str(); }

const char* swb_version(void) {
    return "swb 0.1 (sm_100a; kernels: factorised TMA 2.5D, factorised simple, plain f64, plain f32)";
}

int swb_create(const swb_problem* p, swb_handle** out) {
    if (!p || !out) return fail(SWB_EINVAL, "null argument");
    *out = nullptr;
    for (int d = 0; d < 3; ++d) {
        if (p->shape[d] < 1) return fail(SWB_EINVAL, "grid shape must be positive");
        if (!(p->spacing[d] > 0.0f)) return fail(SWB_EINVAL, "grid spacing must be positive");
    }
    if (p->space_order < 2 || p->space_order % 2 != 0)
        return fail(SWB_EINVAL, "space_order must be an even integer >= 2");
    if (p->space_order > 2 * kMaxH)
        return fail(SWB_EINVAL, "space_order above 24 is not supported");
    if (!(p->dt > 0.0f)) return fail(SWB_EINVAL, "dt must be positive");
    if (!p->m && !p->velocity) return fail(SWB_EINVAL, "m (squared slowness) or the velocity is required");
    if (p->form < 0 || p->form > 4) return fail(SWB_EINVAL, "unknown stencil form");
    if (p->time_block < 0 || p->time_block > 1)
        return fail(SWB_EINVAL, "time_block must be 1: the temporal-blocking kernel (two steps per launch) was "
                                "measured 0.53-0.74x of the single-step kernel on B200 and is retired (DESIGN.md)");
    const int HU = p->space_order / 2;
    const int H = std::max(HU, 1);  // widest halo among u (SO/2), m and damp (1): src/pipeline.cpp:79-88
    const char* dn[3] = {"x", "y", "z"};
    for (int d = 0; d < 3; ++d)
        if (p->shape[d] - 1 - H < H)
            return fail(SWB_EINVAL, "grid extent " + std::to_string(p->shape[d]) + " in " + dn[d] +
                                        " is too small for halo " + std::to_string(H));
    int lo = 0, hi = p->shape[0];
    if (p->slab_hi > 0) {
        lo = p->slab_lo;
        hi = p->slab_hi;
        if (lo < 0 || hi > p->shape[0] || lo >= hi) return fail(SWB_EINVAL, "bad slab range");
        if (hi - lo < HU) return fail(SWB_EINVAL, "slab thinner than SO/2 planes");
    }
    if (p->check_bounds && p->has_source) {
        // RunOptions::check_bounds: the interpreter's first failing access.  The stencil cluster
        // (update interior [H, n-1-H], offsets <= SO/2 into u padded by SO/2; m, damp at offset 0)
        // never leaves the allocation; the source cluster runs after it (src/pipeline.cpp:89-113)
        // and loads u+ then m at the point (its update u+ + dt^2 amp / m, then the store).
        const char* dn3[3] = {"x", "y", "z"};
        const int halo_u = HU, halo_m = 1;
        for (int f = 0; f < 2; ++f) {
            const int hf = f == 0 ? halo_u : halo_m;
            for (int d = 0; d < 3; ++d)
                if (p->source[d] + hf < 0 || p->source[d] + hf >= p->shape[d] + 2 * hf)
                    return fail(SWB_ERANGE, std::string("access to ") + (f == 0 ? "u" : "m") +
                                                " leaves the allocation in " + dn3[d] + " at step 0");
        }
    }
    if (p->check_bounds)
        for (int r = 0; r < p->n_receivers; ++r)  // receivers (an addition) sample u at offset 0
            for (int d = 0; d < 3; ++d)
                if (p->receivers[3 * r + d] + HU < 0 || p->receivers[3 * r + d] + HU >= p->shape[d] + 2 * HU)
                    return fail(SWB_ERANGE, "receiver " + std::to_string(r) + " access to u leaves the allocation");
    if (p->has_source) {
        for (int d = 0; d < 3; ++d)
            if (p->source[d] < HU || p->source[d] > p->shape[d] - 1 - HU)
                return fail(SWB_EINVAL, "source point must lie in the updatable interior");
        if (!p->wavelet || p->wavelet_len < 1)
            return fail(SWB_EINVAL, "source wavelet missing");
    }
    if (p->n_receivers < 0 || (p->n_receivers > 0 && !p->receivers))
        return fail(SWB_EINVAL, "bad receiver list");
    if (p->n_coord_receivers < 0 || (p->n_coord_receivers > 0 && !p->coord_receivers))
        return fail(SWB_EINVAL, "bad coordinate receiver list");
    for (int r = 0; r < p->n_receivers; ++r)
        for (int d = 0; d < 3; ++d)
            if (p->receivers[3 * r + d] < 0 || p->receivers[3 * r + d] >= p->shape[d])
                return fail(SWB_EINVAL, "receiver " + std::to_string(r) + " lies outside the grid");
    int rc = setup_device(p->device);
    if (rc) return rc;

    auto* h = new swb_handle();
    h->device = p->device;
    h->n0 = p->shape[0];
    h->n1 = p->shape[1];
    h->n2 = p->shape[2];
    h->so = p->space_order;
    h->HU = HU;
    h->H = H;
    h->P2 = (h->n2 + 31) / 32 * 32;
    h->lo = lo;
    h->hi = hi;
    h->gb = lo > 0 ? HU : 0;
    h->ga = hi < h->n0 ? HU : 0;
    h->nl0 = (hi - lo) + h->gb + h->ga;
    h->xg_off = lo - h->gb;
    h->plane = static_cast<long long>(h->n1) * h->P2;
    h->level_floats = h->plane * h->nl0;
    h->form = p->form;

    auto cleanup = [&](int code) {
        swb_destroy(h);
        return code;
    };
#define SWB_CUDA_C(call)                                                                   \
    do {                                                                                   \
        cudaError_t e_ = (call);                                                           \
        if (e_ != cudaSuccess)                                                             \
            return cleanup(fail(SWB_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e_))); \
    } while (0)

    const bool prof = std::getenv("SWB_PROFILE_CREATE") != nullptr;  // development timing
    auto now = [] { return std::chrono::steady_clock::now(); };
    auto t_last = now();
    auto mark = [&](const char* what) {
        if (!prof) return;
        cudaStreamSynchronize(h->stream);
        const auto t = now();
        std::fprintf(stderr, "swb_create %-24s %8.3f ms\n", what,
                     std::chrono::duration<double, std::milli>(t - t_last).count());
        t_last = t;
    };
    SWB_CUDA_C(cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking));
    mark("stream");
    SWB_CUDA_C(cudaEventCreate(&h->ev0));
    SWB_CUDA_C(cudaEventCreate(&h->ev1));
    SWB_CUDA_C(pool_alloc(h->device, reinterpret_cast<void**>(&h->u), sizeof(float) * 3 * h->level_floats));
    SWB_CUDA_C(pool_alloc(h->device, reinterpret_cast<void**>(&h->m), sizeof(float) * h->level_floats));
    SWB_CUDA_C(pool_alloc(h->device, reinterpret_cast<void**>(&h->damp), sizeof(float) * h->level_floats));
    SWB_CUDA_C(cudaMemsetAsync(h->u, 0, sizeof(float) * 3 * h->level_floats, h->stream));
    SWB_CUDA_C(cudaMemsetAsync(h->m, 0, sizeof(float) * h->level_floats, h->stream));
    SWB_CUDA_C(cudaMemsetAsync(h->damp, 0, sizeof(float) * h->level_floats, h->stream));
    SWB_CUDA_C(hbuf_alloc(h, &h->d_ring, 3 * sizeof(unsigned)));
    SWB_CUDA_C(hbuf_alloc(h, &h->d_flags, 2 * sizeof(unsigned long long)));
    SWB_CUDA_C(cudaMemsetAsync(h->d_flags, 0, 2 * sizeof(unsigned long long), h->stream));
    SWB_CUDA_C(hbuf_alloc(h, &h->d_err, sizeof(unsigned)));
    SWB_CUDA_C(cudaMemsetAsync(h->d_err, 0, sizeof(unsigned), h->stream));

    mark("malloc+memset");
    // m / damp for every local plane (ghost planes included; they are never read).  Uploaded, or
    // computed on the device from the velocity / the taper parameters (bit-identical to
    // WaveProblem::m_data / damp_data, src/wave_model.cpp:16-45).
    const size_t row = sizeof(float) * h->n2;
    const float* m_src = (p->m ? p->m : p->velocity) + static_cast<size_t>(h->xg_off) * h->n1 * h->n2;
    SWB_CUDA_C(cudaMemcpy2DAsync(h->m, sizeof(float) * h->P2, m_src, row, row,
                                 static_cast<size_t>(h->nl0) * h->n1, cudaMemcpyHostToDevice,
                                 h->stream));
    if (!p->m) SWB_CUDA_C(launch_m_from_velocity(h->m, h->level_floats, h->P2, h->n2, h->stream));
    const bool damp_taper = !p->damp && p->damp_max > 0.0f && p->damp_width > 0;
    if (p->damp) {
        const float* d_src = p->damp + static_cast<size_t>(h->xg_off) * h->n1 * h->n2;
        SWB_CUDA_C(cudaMemcpy2DAsync(h->damp, sizeof(float) * h->P2, d_src, row, row,
                                     static_cast<size_t>(h->nl0) * h->n1, cudaMemcpyHostToDevice,
                                     h->stream));
    } else if (damp_taper) {
        SWB_CUDA_C(launch_damp_taper(h->damp, h->nl0, h->n1, h->P2, h->xg_off, h->n0, h->n1, h->n2, p->damp_max,
                                     p->damp_width, h->stream));
    }
    const bool has_damp = p->damp || damp_taper;
    // host values of m / damp at single cells (source scaling, adjoint weights)
    auto m_at = [&](size_t gi) -> float {
        if (p->m) return p->m[gi];
        const float c = p->velocity[gi];
        return 1.0f / (c * c);
    };
    auto damp_at = [&](size_t gi) -> float {
        if (p->damp) return p->damp[gi];
        if (!damp_taper) return 0.0f;
        const int x = static_cast<int>(gi / (static_cast<size_t>(h->n1) * h->n2));
        const int y = static_cast<int>((gi / h->n2) % h->n1), z = static_cast<int>(gi % h->n2);
        const int dist = std::min({x, h->n0 - 1 - x, y, h->n1 - 1 - y, z, h->n2 - 1 - z});
        if (dist >= p->damp_width) return 0.0f;
        return p->damp_max * (1.0f - static_cast<float>(dist) / static_cast<float>(p->damp_width));
    };
    // FD weights: float(c_k) as the interpreter rounds them (src/executor.cpp:136-138).
    std::vector<float> w(static_cast<size_t>(2 * HU + 1));
    if (p->weights) {
        std::memcpy(w.data(), p->weights, sizeof(float) * w.size());
    } else {
        int64_t num[2 * kMaxH + 1], den[2 * kMaxH + 1];
        swb_fd_weights(2, p->space_order, num, den);
        for (size_t i = 0; i < w.size(); ++i)
            w[i] = static_cast<float>(static_cast<double>(num[i]) / static_cast<double>(den[i]));
    }
    // With SO=2 the halo H (=1) equals HU; Coef carries c_0..c_HU.
    coef_from(p, HU, w.data(), h->K);

    // Geometry: update interior [H, n-H) in every dim, intersected with the owned slab.
    Geo& g = h->geo;
    for (int l = 0; l < 3; ++l) g.lev[l] = h->u + l * h->level_floats;
    g.m = h->m;
    g.damp = h->damp;
    g.plane = h->plane;
    g.P2 = h->P2;
    g.n1 = h->n1;
    g.n2 = h->n2;
    g.x0 = std::max(lo, H) - h->xg_off;
    g.x1 = std::min(hi, h->n0 - H) - h->xg_off;
    if (g.x1 < g.x0) g.x1 = g.x0;
    g.y0 = H;
    g.y1 = h->n1 - H;
    g.z0 = H;
    g.z1 = h->n2 - H;
    g.xg_off = h->xg_off;

    // Source / wavelet / receivers
    Ctl& c = h->ctl;
    c.has_src = 0;
    if (p->has_source) {
        h->wavelet_len = p->wavelet_len;
        SWB_CUDA_C(hbuf_alloc(h, &h->d_wavelet, sizeof(float) * p->wavelet_len));
        SWB_CUDA_C(cudaMemcpyAsync(h->d_wavelet, p->wavelet, sizeof(float) * p->wavelet_len,
                                   cudaMemcpyHostToDevice, h->stream));
        if (p->source[0] >= lo && p->source[0] < hi) {
            c.has_src = 1;
            c.src_x = p->source[0] - h->xg_off;
            c.src_y = p->source[1];
            c.src_z = p->source[2];
            c.src_m = m_at((static_cast<size_t>(p->source[0]) * h->n1 + p->source[1]) * h->n2 + p->source[2]);
        }
    }
    c.wavelet = h->d_wavelet;
    c.wavelet_len = h->wavelet_len;
    // Receivers: every sampling point becomes an 8-corner stencil over this slab's planes.
    h->n_rec = p->n_receivers + std::max(0, p->n_coord_receivers);
    std::vector<long long> ridx;
    std::vector<double> rw;
    auto local_index = [&](int x, int y, int z) -> long long {
        if (x < lo || x >= hi) return -1;
        return (x - h->xg_off) * h->plane + static_cast<long long>(y) * h->P2 + z;
    };
    for (int r = 0; r < p->n_receivers; ++r) {
        const int* q = p->receivers + 3 * r;
        if (q[0] >= lo && q[0] < hi) {
            h->rec_owned.push_back(r);
            ridx.push_back(local_index(q[0], q[1], q[2]));
            rw.push_back(1.0);
            for (int c = 1; c < 8; ++c) {
                ridx.push_back(-1);
                rw.push_back(0.0);
            }
        }
    }
    for (int r = 0; r < std::max(0, p->n_coord_receivers); ++r) {
        const double* X = p->coord_receivers + 3 * r;
        int i0[3];
        double f[3];
        for (int d = 0; d < 3; ++d) {
            const double hd = static_cast<double>(p->spacing[d]);
            const double gx = X[d] / hd;
            if (!(gx >= 0.0) || gx > static_cast<double>(p->shape[d] - 1))
                return cleanup(fail(SWB_EINVAL, "receiver coordinate " + std::to_string(r) + " lies outside the grid"));
            int i = static_cast<int>(std::floor(gx));
            if (i >= p->shape[d] - 1) i = p->shape[d] - 2;
            i0[d] = i;
            f[d] = gx - static_cast<double>(i);
        }
        std::vector<long long> ci(8);
        std::vector<double> cw(8);
        bool any = false;
        int c = 0;
        for (int a = 0; a < 2; ++a)
            for (int b = 0; b < 2; ++b)
                for (int e = 0; e < 2; ++e, ++c) {
                    const double wa = a ? f[0] : 1.0 - f[0], wb = b ? f[1] : 1.0 - f[1], we = e ? f[2] : 1.0 - f[2];
                    cw[c] = (wa * wb) * we;
                    ci[c] = local_index(i0[0] + a, i0[1] + b, i0[2] + e);
                    any |= ci[c] >= 0;
                }
        if (any) {
            h->rec_owned.push_back(p->n_receivers + r);
            ridx.insert(ridx.end(), ci.begin(), ci.end());
            rw.insert(rw.end(), cw.begin(), cw.end());
        }
    }
    if (!ridx.empty()) {
        // adjoint injection weights (swb_apply_adjoint): D^{-1} R^T restricted to the update
        // interior (the forward operator never writes the ring, so it has no adjoint there)
        std::vector<double> iw(rw.size(), 0.0);
        const double dtd = static_cast<double>(p->dt);
        const int Hh = H;
        for (size_t q = 0; q < ridx.size(); ++q) {
            if (ridx[q] < 0) continue;
            const long long j = ridx[q];
            const int lx = static_cast<int>(j / h->plane) + h->xg_off;
            const int y = static_cast<int>((j % h->plane) / h->P2), z = static_cast<int>(j % h->P2);
            if (lx < Hh || lx > h->n0 - 1 - Hh || y < Hh || y > h->n1 - 1 - Hh || z < Hh || z > h->n2 - 1 - Hh)
                continue;
            const size_t gi = (static_cast<size_t>(lx) * h->n1 + y) * h->n2 + z;
            const double mm = m_at(gi), dd = damp_at(gi);
            iw[q] = rw[q] / (mm + 0.5 * dd * dtd);
        }
        SWB_CUDA_C(hbuf_alloc(h, &h->d_inj_w, sizeof(double) * iw.size()));
        SWB_CUDA_C(cudaMemcpyAsync(h->d_inj_w, iw.data(), sizeof(double) * iw.size(), cudaMemcpyHostToDevice,
                                   h->stream));
        SWB_CUDA_C(hbuf_alloc(h, &h->d_rec_idx, sizeof(long long) * ridx.size()));
        SWB_CUDA_C(hbuf_alloc(h, &h->d_rec_w, sizeof(double) * rw.size()));
        SWB_CUDA_C(cudaMemcpyAsync(h->d_rec_idx, ridx.data(), sizeof(long long) * ridx.size(),
                                   cudaMemcpyHostToDevice, h->stream));
        SWB_CUDA_C(cudaMemcpyAsync(h->d_rec_w, rw.data(), sizeof(double) * rw.size(), cudaMemcpyHostToDevice,
                                   h->stream));
    }
    mark("H2D m/damp, weights, rec");
    // Adjoint output sampler at the source point (owned slab only).
    if (c.has_src) {
        const size_t gi = (static_cast<size_t>(p->source[0]) * h->n1 + p->source[1]) * h->n2 + p->source[2];
        const double mm = m_at(gi), dd = damp_at(gi), dtd = static_cast<double>(p->dt);
        std::vector<long long> si(8, -1);
        std::vector<double> sw(8, 0.0);
        si[0] = local_index(p->source[0], p->source[1], p->source[2]);
        sw[0] = ((dtd * dtd) * (mm + 0.5 * dd * dtd)) / mm;
        SWB_CUDA_C(hbuf_alloc(h, &h->d_src_idx, sizeof(long long) * 8));
        SWB_CUDA_C(hbuf_alloc(h, &h->d_src_w, sizeof(double) * 8));
        SWB_CUDA_C(cudaMemcpyAsync(h->d_src_idx, si.data(), sizeof(long long) * 8, cudaMemcpyHostToDevice, h->stream));
        SWB_CUDA_C(cudaMemcpyAsync(h->d_src_w, sw.data(), sizeof(double) * 8, cudaMemcpyHostToDevice, h->stream));
    }
    mark("adjoint sampler");
    // Kernel choice: the TMA 2.5D kernel for the factorised form when the plan fits.
    if (h->form == SWB_FORM_FACTORISED) {
        int sms = device_sm_count();  // (current device = h->device, set by setup_device)
        if (const char* cap = std::getenv("SWB_MAX_CTAS")) sms = std::max(1, std::min(sms, std::atoi(cap)));
        h->plan = tma_plan(HU, g, sms);
        if (h->plan.ok && h->K.iso) {
            SWB_CUDA_C(tma_make_maps(h->plan, g, h->nl0, h->maps));
            const size_t nflags = static_cast<size_t>(h->plan.columns) * std::max(0, g.x1 - g.x0);
            SWB_CUDA_C(hbuf_alloc(h, &h->d_dflag, std::max<size_t>(nflags, 1)));
            SWB_CUDA_C(cudaMemsetAsync(h->d_dflag, 0, std::max<size_t>(nflags, 1), h->stream));
            if (has_damp) SWB_CUDA_C(tma_damp_flags_device(h->plan, g, h->d_dflag, h->stream));
            h->plan.dflag = h->d_dflag;
            h->use_tma = true;
            // K1 reads m and damp only as the update coefficients B = 1/(m+g), A = (m-g)/(m+g):
            // transform them in place (after the damp flags above, same stream)
            SWB_CUDA_C(tma_update_coefs(h->m, h->damp, h->level_floats, h->K.half_dt, h->P2, h->n1, h->n2,
                                            h->xg_off, h->stream));
        }
    }
    h->stats.kernel_variant = h->use_tma ? h->plan.variant : 100 + h->form;
    if (std::getenv("SWB_TRACE") && h->use_tma) {
        SWB_CUDA_C(cudaMalloc(&h->d_trace, sizeof(unsigned long long) * 2 * 8 * 1024));
        SWB_CUDA_C(cudaMemset(h->d_trace, 0, sizeof(unsigned long long) * 2 * 8 * 1024));
        h->ctl.trace = h->d_trace;
    }
    h->stats.launch_steps = 1;
    compute_peer_ranges(h);
    mark("plan+maps+dflags");
    SWB_CUDA_C(cudaStreamSynchronize(h->stream));
    *out = h;
#undef SWB_CUDA_C
    return SWB_OK;
}

int swb_set_level(swb_handle* h, int level, const float* src) {
    if (!h || !src || level < 0 || level > 2) return fail(SWB_EINVAL, "bad set_level arguments");
    if (h->pending) return fail(SWB_EINVAL, "an asynchronous apply is pending");
    SWB_CUDA(cudaSetDevice(h->device));
    const size_t row = sizeof(float) * h->n2;
    const float* s = src + static_cast<size_t>(h->xg_off) * h->n1 * h->n2;
    SWB_CUDA(cudaMemcpy2DAsync(h->u + level * h->level_floats, sizeof(float) * h->P2, s, row, row,
                               static_cast<size_t>(h->nl0) * h->n1, cudaMemcpyHostToDevice,
                               h->stream));
    h->ring_dirty = true;
    SWB_CUDA(cudaStreamSynchronize(h->stream));
    return SWB_OK;
}

int swb_get_level(swb_handle* h, int level, float* dst) {
    if (!h || !dst || level < 0 || level > 2) return fail(SWB_EINVAL, "bad get_level arguments");
    if (h->pending) return fail(SWB_EINVAL, "an asynchronous apply is pending");
    SWB_CUDA(cudaSetDevice(h->device));
    const size_t row = sizeof(float) * h->n2;
    float* d = dst + static_cast<size_t>(h->lo) * h->n1 * h->n2;
    SWB_CUDA(cudaMemcpy2DAsync(d, row, h->u + level * h->level_floats + h->gb * h->plane,
                               sizeof(float) * h->P2, row,
                               static_cast<size_t>(h->hi - h->lo) * h->n1, cudaMemcpyDeviceToHost,
                               h->stream));
    SWB_CUDA(cudaStreamSynchronize(h->stream));
    return SWB_OK;
}

int swb_get_level_padded(swb_handle* h, int level, float* dst, int halo) {
    if (!h || !dst || level < 0 || level > 2 || halo < 0) return fail(SWB_EINVAL, "bad get_level_padded arguments");
    if (h->pending) return fail(SWB_EINVAL, "an asynchronous apply is pending");
    SWB_CUDA(cudaSetDevice(h->device));
    // owned planes [lo, hi) of the level -> the padded host block at (lo + halo, halo, halo)
    cudaMemcpy3DParms cp{};
    cp.srcPtr = make_cudaPitchedPtr(h->u + level * h->level_floats + h->gb * h->plane, sizeof(float) * h->P2,
                                    sizeof(float) * h->n2, h->n1);
    cp.dstPtr = make_cudaPitchedPtr(dst, sizeof(float) * (h->n2 + 2 * halo), sizeof(float) * (h->n2 + 2 * halo),
                                    h->n1 + 2 * halo);
    cp.dstPos = make_cudaPos(sizeof(float) * halo, halo, h->lo + halo);
    cp.extent = make_cudaExtent(sizeof(float) * h->n2, h->n1, h->hi - h->lo);
    cp.kind = cudaMemcpyDeviceToHost;
    SWB_CUDA(cudaMemcpy3DAsync(&cp, h->stream));
    SWB_CUDA(cudaStreamSynchronize(h->stream));
    return SWB_OK;
}

int swb_apply_async(swb_handle* h, int step0, int nt) {
    if (!h) return fail(SWB_EINVAL, "null handle");
    if (h->pending) return fail(SWB_EINVAL, "an asynchronous apply is already pending");
    if (step0 < 0 || nt < 0) return fail(SWB_EINVAL, "steps must be non-negative");
    if (h->ctl.wavelet && step0 + nt > h->wavelet_len)
        return fail(SWB_EINVAL, "source wavelet shorter than the number of steps");
    SWB_CUDA(cudaSetDevice(h->device));
    int rc = ensure_smax(h, nt);
    if (rc) return rc;
    rc = ensure_traces(h, nt);
    if (rc) return rc;
    rc = refresh_ring(h);
    if (rc) return rc;
    if (nt > 0) SWB_CUDA(cudaMemsetAsync(h->d_smax, 0, sizeof(unsigned) * nt, h->stream));
    h->launches = 0;
    h->ctl.smax = h->d_smax;
    SWB_CUDA(cudaEventRecord(h->ev0, h->stream));
    rc = enqueue_steps(h, step0, nt);
    if (rc) return rc;
    SWB_CUDA(cudaEventRecord(h->ev1, h->stream));
    h->pend_step0 = step0;
    h->pend_nt = nt;
    h->pending = true;
    return SWB_OK;
}

int swb_collect(swb_handle* h, float* step_max_abs, int32_t* first_bad_step, float* rec_traces) {
    if (!h) return fail(SWB_EINVAL, "null handle");
    if (!h->pending) return fail(SWB_EINVAL, "no apply pending");
    SWB_CUDA(cudaSetDevice(h->device));
    h->pending = false;
    const int nt = h->pend_nt, step0 = h->pend_step0;
    SWB_CUDA(cudaStreamSynchronize(h->stream));
    float ms = 0.f;
    cudaEventElapsedTime(&ms, h->ev0, h->ev1);
    h->stats.device_ms = ms;
    h->stats.kernel_launches = h->launches;
    const uint64_t per_step =
        static_cast<uint64_t>(std::max(0, h->geo.x1 - h->geo.x0)) *
            static_cast<uint64_t>(h->geo.y1 - h->geo.y0) * static_cast<uint64_t>(h->geo.z1 - h->geo.z0) +
        (h->ctl.has_src ? 1u : 0u);
    h->stats.point_updates += per_step * static_cast<uint64_t>(nt);
    unsigned herr = 0;
    SWB_CUDA(cudaMemcpy(&herr, h->d_err, sizeof herr, cudaMemcpyDeviceToHost));
    if (herr) {
        cudaMemset(h->d_err, 0, sizeof herr);
        return fail(SWB_ECUDA, "halo exchange timed out waiting for a neighbour slab");
    }
    std::vector<unsigned> smax(static_cast<size_t>(nt)), ring(3);
    if (nt > 0)
        SWB_CUDA(cudaMemcpy(smax.data(), h->d_smax, sizeof(unsigned) * nt, cudaMemcpyDeviceToHost));
    SWB_CUDA(cudaMemcpy(ring.data(), h->d_ring, sizeof(unsigned) * 3, cudaMemcpyDeviceToHost));
    int bad = -1;
    for (int i = 0; i < nt; ++i) {
        const unsigned bits = std::max(smax[i], ring[(step0 + i + 1) % 3]);
        float v;
        if (bits >= 0x7f800000u) {
            v = std::nanf("");
            if (bad < 0) bad = step0 + i;
        } else {
            std::memcpy(&v, &bits, sizeof v);
        }
        if (step_max_abs) step_max_abs[i] = v;
    }
    if (first_bad_step) *first_bad_step = bad;
    if (rec_traces && h->n_rec > 0) {
        const int owned = static_cast<int>(h->rec_owned.size());
        std::memset(rec_traces, 0, sizeof(float) * static_cast<size_t>(nt) * h->n_rec);
        if (owned > 0 && nt > 0) {
            std::vector<float> t(static_cast<size_t>(nt) * owned);
            SWB_CUDA(cudaMemcpy(t.data(), h->d_traces, sizeof(float) * t.size(),
                                cudaMemcpyDeviceToHost));
            for (int i = 0; i < nt; ++i)
                for (int r = 0; r < owned; ++r)
                    rec_traces[static_cast<size_t>(i) * h->n_rec + h->rec_owned[r]] =
                        t[static_cast<size_t>(i) * owned + r];
        }
    }
    if (bad >= 0)
        return fail(SWB_EUNSTABLE,
                    "non-finite wave field at step " + std::to_string(bad) + " (unstable dt?)");
    return SWB_OK;
}

int swb_apply(swb_handle* h, int step0, int nt, float* step_max_abs, int32_t* first_bad_step,
              float* rec_traces) {
    int rc = swb_apply_async(h, step0, nt);
    if (rc) return rc;
    return swb_collect(h, step_max_abs, first_bad_step, rec_traces);
}

int swb_apply_adjoint(swb_handle* h, int nt, const float* rec_data, float* src_trace, float* step_max_abs,
                      int32_t* first_bad_step) {
    if (!h) return fail(SWB_EINVAL, "null handle");
    if (h->pending) return fail(SWB_EINVAL, "an asynchronous apply is pending");
    if (nt < 0) return fail(SWB_EINVAL, "steps must be non-negative");
    if (linked(h)) return fail(SWB_EINVAL, "the adjoint runs on a single-domain handle (not on linked slabs)");
    if (!h->ctl.has_src || !h->d_src_idx) return fail(SWB_EINVAL, "the adjoint samples at the source point: the problem needs a source");
    if (h->n_rec <= 0 || !rec_data) return fail(SWB_EINVAL, "the adjoint injects receiver data: receivers are required");
    SWB_CUDA(cudaSetDevice(h->device));
    const int owned = static_cast<int>(h->rec_owned.size());
    if (nt > h->adj_cap) {
        if (h->d_adj) cudaFree(h->d_adj);
        if (h->d_src_trace) cudaFree(h->d_src_trace);
        h->d_adj = nullptr;
        h->d_src_trace = nullptr;
        SWB_CUDA(cudaMalloc(&h->d_adj, sizeof(float) * static_cast<size_t>(std::max(nt, 1)) * std::max(owned, 1)));
        SWB_CUDA(cudaMalloc(&h->d_src_trace, sizeof(float) * static_cast<size_t>(std::max(nt, 1))));
        h->adj_cap = nt;
    }
    int rc = ensure_smax(h, nt);
    if (rc) return rc;
    {
        std::vector<float> gathered(static_cast<size_t>(nt) * owned);
        for (int i = 0; i < nt; ++i)
            for (int r = 0; r < owned; ++r)
                gathered[static_cast<size_t>(i) * owned + r] = rec_data[static_cast<size_t>(i) * h->n_rec + h->rec_owned[r]];
        if (!gathered.empty())
            SWB_CUDA(cudaMemcpyAsync(h->d_adj, gathered.data(), sizeof(float) * gathered.size(),
                                     cudaMemcpyHostToDevice, h->stream));
        // adjoint state starts at zero (all levels, ring included)
        SWB_CUDA(cudaMemsetAsync(h->u, 0, sizeof(float) * 3 * h->level_floats, h->stream));
        SWB_CUDA(cudaMemsetAsync(h->d_ring, 0, 3 * sizeof(unsigned), h->stream));
        h->ring_dirty = false;
        if (nt > 0) SWB_CUDA(cudaMemsetAsync(h->d_smax, 0, sizeof(unsigned) * nt, h->stream));
        h->ctl.smax = h->d_smax;
        h->launches = 0;
        SWB_CUDA(cudaEventRecord(h->ev0, h->stream));
        for (int sp = 0; sp < nt; ++sp) {
            const int k = nt - sp;  // z[k] = stencil(z[k+1], z[k+2]) + D^-1 R^T d[k-1]
            Ctl c = h->ctl;
            c.has_src = 0;
            c.step = sp;
            c.slot = sp;
            c.err = h->d_err;
            c.ghost_lo_end = 0;
            c.ghost_hi_begin = INT_MAX;
            if (h->use_tma) {
                SWB_CUDA(launch_tma(h->plan, h->maps, h->geo, h->K, c, h->peer, h->stream));
            } else {
                const int form = h->form == SWB_FORM_PLAIN_F64   ? 1
                                 : h->form == SWB_FORM_PLAIN_F32 ? 2
                                 : h->form == SWB_FORM_FACTORISED_SIMPLE_F32C ? 3
                                                                         : 0;
                SWB_CUDA(launch_simple(h->H, form, h->geo, h->K, c, h->peer, h->stream));
            }
            float* un = h->u + ((sp + 1) % 3) * h->level_floats;
            SWB_CUDA(launch_inject(un, h->d_rec_idx, h->d_inj_w, owned, h->d_adj + static_cast<size_t>(k - 1) * owned,
                                   h->stream));
            SWB_CUDA(launch_samplers(un, h->d_src_idx, h->d_src_w, 1, h->d_src_trace + (k - 1), h->stream));
            h->launches += 3;
        }
        SWB_CUDA(cudaEventRecord(h->ev1, h->stream));
    }
    SWB_CUDA(cudaStreamSynchronize(h->stream));
    float ms = 0.f;
    cudaEventElapsedTime(&ms, h->ev0, h->ev1);
    h->stats.device_ms = ms;
    h->stats.kernel_launches = h->launches;
    h->ring_dirty = true;
    unsigned herr = 0;
    SWB_CUDA(cudaMemcpy(&herr, h->d_err, sizeof herr, cudaMemcpyDeviceToHost));
    if (herr) {
        cudaMemset(h->d_err, 0, sizeof herr);
        return fail(SWB_ECUDA, "device wait timed out");
    }
    std::vector<unsigned> smax(static_cast<size_t>(nt));
    if (nt > 0) SWB_CUDA(cudaMemcpy(smax.data(), h->d_smax, sizeof(unsigned) * nt, cudaMemcpyDeviceToHost));
    if (src_trace && nt > 0)
        SWB_CUDA(cudaMemcpy(src_trace, h->d_src_trace, sizeof(float) * nt, cudaMemcpyDeviceToHost));
    int bad = -1;
    for (int i = 0; i < nt; ++i) {
        float v;
        if (smax[i] >= 0x7f800000u) {
            v = std::nanf("");
            if (bad < 0) bad = i;
        } else {
            std::memcpy(&v, &smax[i], sizeof v);
        }
        if (step_max_abs) step_max_abs[i] = v;
    }
    if (first_bad_step) *first_bad_step = bad;
    if (bad >= 0) return fail(SWB_EUNSTABLE, "non-finite adjoint field at adjoint step " + std::to_string(bad));
    return SWB_OK;
}

int swb_apply_snapshots(swb_handle* h, int step0, int nt, int every, float* const* snaps, int n_snaps,
                        float* step_max_abs, int32_t* first_bad_step, float* rec_traces) {
    if (!h) return fail(SWB_EINVAL, "null handle");
    if (h->pending) return fail(SWB_EINVAL, "an asynchronous apply is already pending");
    if (step0 < 0 || nt < 0 || every < 1) return fail(SWB_EINVAL, "steps must be non-negative and every >= 1");
    if (n_snaps != nt / every || (n_snaps > 0 && !snaps))
        return fail(SWB_EINVAL, "need one snapshot buffer per `every` steps (nt / every of them)");
    if (h->ctl.wavelet && step0 + nt > h->wavelet_len)
        return fail(SWB_EINVAL, "source wavelet shorter than the number of steps");
    SWB_CUDA(cudaSetDevice(h->device));
    int rc = ensure_smax(h, nt);
    if (rc) return rc;
    rc = ensure_traces(h, nt);
    if (rc) return rc;
    rc = refresh_ring(h);
    if (rc) return rc;
    const size_t own_floats = static_cast<size_t>(h->hi - h->lo) * h->plane;
    if (n_snaps > 0 && !h->s_d2d) {
        SWB_CUDA(cudaStreamCreateWithFlags(&h->s_d2d, cudaStreamNonBlocking));
        SWB_CUDA(cudaStreamCreateWithFlags(&h->s_d2h, cudaStreamNonBlocking));
        SWB_CUDA(cudaEventCreateWithFlags(&h->ev_step, cudaEventDisableTiming));
        for (int j = 0; j < swb_handle::kSnapSlots; ++j) {
            SWB_CUDA(cudaEventCreateWithFlags(&h->ev_d2d[j], cudaEventDisableTiming));
            SWB_CUDA(cudaEventCreateWithFlags(&h->ev_d2h[j], cudaEventDisableTiming));
            SWB_CUDA(cudaMalloc(&h->d_stage[j], sizeof(float) * own_floats));
        }
    }
    if (nt > 0) SWB_CUDA(cudaMemsetAsync(h->d_smax, 0, sizeof(unsigned) * nt, h->stream));
    h->launches = 0;
    h->ctl.smax = h->d_smax;
    SWB_CUDA(cudaEventRecord(h->ev0, h->stream));
    const size_t row = sizeof(float) * h->n2;
    int done = 0;
    for (int i = 0; i < n_snaps; ++i) {
        // steps of this interval; the first two may run before the previous snapshot's device
        // copy is complete (the level it copies is overwritten by the third step after it)
        const int a = std::min(2, every);
        rc = enqueue_steps(h, step0 + done, a, done);
        if (rc) return rc;
        if (i > 0) SWB_CUDA(cudaStreamWaitEvent(h->stream, h->ev_d2d[(i - 1) % swb_handle::kSnapSlots], 0));
        if (every > a) {
            rc = enqueue_steps(h, step0 + done + a, every - a, done + a);
            if (rc) return rc;
        }
        done += every;
        const int lev = (step0 + done) % 3;  // newest level after step step0 + done - 1
        const int j = i % swb_handle::kSnapSlots;
        SWB_CUDA(cudaEventRecord(h->ev_step, h->stream));
        SWB_CUDA(cudaStreamWaitEvent(h->s_d2d, h->ev_step, 0));
        if (i >= swb_handle::kSnapSlots) SWB_CUDA(cudaStreamWaitEvent(h->s_d2d, h->ev_d2h[j], 0));
        SWB_CUDA(cudaMemcpyAsync(h->d_stage[j], h->u + lev * h->level_floats + h->gb * h->plane,
                                 sizeof(float) * own_floats, cudaMemcpyDeviceToDevice, h->s_d2d));
        SWB_CUDA(cudaEventRecord(h->ev_d2d[j], h->s_d2d));
        SWB_CUDA(cudaStreamWaitEvent(h->s_d2h, h->ev_d2d[j], 0));
        SWB_CUDA(cudaMemcpy2DAsync(snaps[i] + static_cast<size_t>(h->lo) * h->n1 * h->n2, row, h->d_stage[j],
                                   sizeof(float) * h->P2, row, static_cast<size_t>(h->hi - h->lo) * h->n1,
                                   cudaMemcpyDeviceToHost, h->s_d2h));
        SWB_CUDA(cudaEventRecord(h->ev_d2h[j], h->s_d2h));
    }
    if (n_snaps > 0) SWB_CUDA(cudaStreamWaitEvent(h->stream, h->ev_d2d[(n_snaps - 1) % swb_handle::kSnapSlots], 0));
    if (nt > done) {
        rc = enqueue_steps(h, step0 + done, nt - done, done);
        if (rc) return rc;
    }
    SWB_CUDA(cudaEventRecord(h->ev1, h->stream));
    h->pend_step0 = step0;
    h->pend_nt = nt;
    h->pending = true;
    if (h->s_d2h) SWB_CUDA(cudaStreamSynchronize(h->s_d2h));
    return swb_collect(h, step_max_abs, first_bad_step, rec_traces);
}

void* swb_stream(swb_handle* h) { return h ? static_cast<void*>(h->stream) : nullptr; }

// Debug (SWB_TRACE=1): copy the per-CTA timestamps of the last stencil launch.
int swb_debug_trace(swb_handle* h, unsigned long long* out, int max_ctas) {
    if (!h || !h->d_trace) return fail(SWB_EINVAL, "tracing not enabled (set SWB_TRACE=1)");
    SWB_CUDA(cudaStreamSynchronize(h->stream));
    const int n = std::min(max_ctas, 1024);
    for (int par = 0; par < 2; ++par)
        SWB_CUDA(cudaMemcpy(out + static_cast<size_t>(par) * 8 * n, h->d_trace + static_cast<size_t>(par) * 8 * 1024,
                            sizeof(unsigned long long) * 8 * n, cudaMemcpyDeviceToHost));
    return h->plan.grid;
}

int swb_get_stats(swb_handle* h, swb_stats* out) {
    if (!h || !out) return fail(SWB_EINVAL, "null argument");
    h->stats.peer_lo = h->lo_remote ? h->peer_dev_lo : -1;
    h->stats.peer_hi = h->hi_remote ? h->peer_dev_hi : -1;
    h->stats.fused_lo = h->fused_lo;
    h->stats.fused_hi = h->fused_hi;
    h->stats.grid = h->use_tma ? h->plan.grid : 0;
    *out = h->stats;
    return SWB_OK;
}

int swb_destroy(swb_handle* h) {
    if (!h) return SWB_OK;
    cudaSetDevice(h->device);
    if (h->stream) cudaStreamSynchronize(h->stream);
    // snapshot copies may still read u (an apply_snapshots that returned early on an error)
    if (h->s_d2d) cudaStreamSynchronize(h->s_d2d);
    if (h->s_d2h) cudaStreamSynchronize(h->s_d2h);
    if (h->ipc_lo_u) cudaIpcCloseMemHandle(h->ipc_lo_u);
    if (h->ipc_hi_u) cudaIpcCloseMemHandle(h->ipc_hi_u);
    if (h->ipc_lo_f) cudaIpcCloseMemHandle(h->ipc_lo_f);
    if (h->ipc_hi_f) cudaIpcCloseMemHandle(h->ipc_hi_f);
    // the big buffers go back to the pool (the stream is idle: synchronised above)
    pool_free(h->device, h->u, sizeof(float) * 3 * h->level_floats, h->exported);
    pool_free(h->device, h->m, sizeof(float) * h->level_floats);
    pool_free(h->device, h->damp, sizeof(float) * h->level_floats);
    // (the step counters are IPC-exported with u: never recycled either)
    for (const auto& b : h->hbufs)
        pool_free(h->device, b.first, b.second, h->exported && b.first == static_cast<void*>(h->d_flags));
    h->hbufs.clear();
    for (void* q : {static_cast<void*>(h->d_adj), static_cast<void*>(h->d_src_trace),
                    static_cast<void*>(h->d_trace)})
        if (q) cudaFree(q);
    for (int j = 0; j < swb_handle::kSnapSlots; ++j) {
        if (h->d_stage[j]) cudaFree(h->d_stage[j]);
        if (h->ev_d2d[j]) cudaEventDestroy(h->ev_d2d[j]);
        if (h->ev_d2h[j]) cudaEventDestroy(h->ev_d2h[j]);
    }
    if (h->ev_step) cudaEventDestroy(h->ev_step);
    if (h->s_d2d) cudaStreamDestroy(h->s_d2d);
    if (h->s_d2h) cudaStreamDestroy(h->s_d2h);
    if (h->ev0) cudaEventDestroy(h->ev0);
    if (h->ev1) cudaEventDestroy(h->ev1);
    if (h->stream) cudaStreamDestroy(h->stream);
    delete h;
    return SWB_OK;
}

// ---- halo linking ----------------------------------------------------------------------

int swb_link_local(swb_handle* lower, swb_handle* upper) {
    if (!lower || !upper) return fail(SWB_EINVAL, "null handle");
    if (lower->hi != upper->lo || lower->n1 != upper->n1 || lower->n2 != upper->n2 ||
        lower->HU != upper->HU)
        return fail(SWB_EINVAL, "handles are not adjacent slabs of one grid");
    if (lower->device != upper->device) {
        int can = 0;
        SWB_CUDA(cudaDeviceCanAccessPeer(&can, lower->device, upper->device));
        if (!can) return fail(SWB_ECUDA, "no peer access between the two devices");
        cudaSetDevice(lower->device);
        cudaError_t e = cudaDeviceEnablePeerAccess(upper->device, 0);
        if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled)
            return fail(SWB_ECUDA, cudaGetErrorString(e));
        cudaGetLastError();
        cudaSetDevice(upper->device);
        e = cudaDeviceEnablePeerAccess(lower->device, 0);
        if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled)
            return fail(SWB_ECUDA, cudaGetErrorString(e));
        cudaGetLastError();
    }
    for (int l = 0; l < 3; ++l) {
        lower->peer.hi_lev[l] = upper->u + l * upper->level_floats;
        upper->peer.lo_lev[l] = lower->u + l * lower->level_floats;
    }
    lower->peer.hi_shift = lower->xg_off - upper->xg_off;
    upper->peer.lo_shift = upper->xg_off - lower->xg_off;
    lower->hi_remote = upper->d_flags + 0;
    upper->lo_remote = lower->d_flags + 1;
    // Same-device slabs run their persistent kernels concurrently on one GPU: in-kernel waits
    // are only safe if both grids fit at once, so they are opt-in there (tests cap the grid
    // with SWB_MAX_CTAS).  Across devices they are always safe.
    const bool same_dev = lower->device == upper->device;
    const int fused = fused_capable(lower) && fused_capable(upper) &&
                      (!same_dev || std::getenv("SWB_FUSED_SAME_DEVICE") != nullptr);
    lower->fused_hi = upper->fused_lo = fused;
    lower->peer_dev_hi = upper->device;
    upper->peer_dev_lo = lower->device;
    lower->nb_grid_hi = upper->plan.grid;
    upper->nb_grid_lo = lower->plan.grid;
    compute_peer_ranges(lower);
    compute_peer_ranges(upper);
    return SWB_OK;
}

int swb_export_ghosts(swb_handle* h, void* blob, size_t* blob_len) {
    if (!h || !blob_len) return fail(SWB_EINVAL, "null argument");
    if (!blob || *blob_len < sizeof(IpcBlob)) {
        *blob_len = sizeof(IpcBlob);
        return blob ? fail(SWB_EINVAL, "blob buffer too small") : SWB_OK;
    }
    SWB_CUDA(cudaSetDevice(h->device));
    IpcBlob b{};
    b.magic = kBlobMagic;
    b.xg_off = h->xg_off;
    b.nl0 = h->nl0;
    b.n1 = h->n1;
    b.n2 = h->n2;
    b.P2 = h->P2;
    b.H = h->HU;
    b.fused_capable = fused_capable(h) ? 1 : 0;
    {
        cudaDeviceProp prop{};
        SWB_CUDA(cudaGetDeviceProperties(&prop, h->device));
        std::memcpy(b.uuid, prop.uuid.bytes, 16);
    }
    b.grid = h->plan.grid;
    b.level_floats = h->level_floats;
    SWB_CUDA(cudaIpcGetMemHandle(&b.u_handle, h->u));
    h->exported = true;
    SWB_CUDA(cudaIpcGetMemHandle(&b.flag_handle, h->d_flags));
    std::memcpy(blob, &b, sizeof b);
    *blob_len = sizeof b;
    return SWB_OK;
}

int swb_link_neighbours(swb_handle* h, const void* lower_blob, size_t lower_len,
                        const void* upper_blob, size_t upper_len) {
    if (!h) return fail(SWB_EINVAL, "null handle");
    SWB_CUDA(cudaSetDevice(h->device));
    auto open = [&](const void* blob, size_t len, IpcBlob& b, void** u, void** f) -> int {
        if (len < sizeof(IpcBlob)) return fail(SWB_EINVAL, "short neighbour blob");
        std::memcpy(&b, blob, sizeof b);
        if (b.magic != kBlobMagic || b.n1 != h->n1 || b.n2 != h->n2 || b.P2 != h->P2 || b.H != h->HU)
            return fail(SWB_EINVAL, "neighbour blob does not describe a slab of this grid");
        SWB_CUDA(cudaIpcOpenMemHandle(u, b.u_handle, cudaIpcMemLazyEnablePeerAccess));
        SWB_CUDA(cudaIpcOpenMemHandle(f, b.flag_handle, cudaIpcMemLazyEnablePeerAccess));
        return SWB_OK;
    };
    if (lower_blob && lower_len) {
        IpcBlob b;
        int rc = open(lower_blob, lower_len, b, &h->ipc_lo_u, &h->ipc_lo_f);
        if (rc) return rc;
        float* base = static_cast<float*>(h->ipc_lo_u);
        for (int l = 0; l < 3; ++l) h->peer.lo_lev[l] = base + l * b.level_floats;
        h->peer.lo_shift = h->xg_off - b.xg_off;
        h->lo_remote = static_cast<unsigned long long*>(h->ipc_lo_f) + 1;
        h->fused_lo = b.fused_capable && fused_capable(h) &&
                      (!same_device(h->device, b.uuid) || std::getenv("SWB_FUSED_SAME_DEVICE") != nullptr);
        h->nb_grid_lo = b.grid;
        h->peer_dev_lo = device_of_uuid(b.uuid);
    }
    if (upper_blob && upper_len) {
        IpcBlob b;
        int rc = open(upper_blob, upper_len, b, &h->ipc_hi_u, &h->ipc_hi_f);
        if (rc) return rc;
        float* base = static_cast<float*>(h->ipc_hi_u);
        for (int l = 0; l < 3; ++l) h->peer.hi_lev[l] = base + l * b.level_floats;
        h->peer.hi_shift = h->xg_off - b.xg_off;
        h->hi_remote = static_cast<unsigned long long*>(h->ipc_hi_f) + 0;
        h->fused_hi = b.fused_capable && fused_capable(h) &&
                      (!same_device(h->device, b.uuid) || std::getenv("SWB_FUSED_SAME_DEVICE") != nullptr);
        h->nb_grid_hi = b.grid;
        h->peer_dev_hi = device_of_uuid(b.uuid);
    }
    compute_peer_ranges(h);
    return SWB_OK;
}

}  // extern "C"
