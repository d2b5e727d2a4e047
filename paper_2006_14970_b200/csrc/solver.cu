// Host orchestration and the extern "C" boundary (include/fgmatte_b200.h).
//
// A solve is planned on the host (level schedule, coarse/big split, pass
// decomposition, workspace carving -- all O(levels)) and then enqueued on one
// stream: one K4 launch for every image's coarse levels, then, level by level
// from the coarse end, one batched K1/K2 launch and one K3 launch per pass.
#include <cuda_runtime.h>

#include <algorithm>
#include <bit>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <atomic>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/fgmatte_b200.h"
#include "fgm_internal.h"

namespace fgm {
namespace {

thread_local std::string g_err;

struct InvalidArgument : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct RuntimeError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

void ck(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw RuntimeError(std::string(what) + ": " + cudaGetErrorString(e));
}

struct Level {
    int w, h, iters;
};

// MlParams::validate (multilevel.cpp:10-15), same messages.
void validate(const fgm_params* p) {
    if (!p) throw InvalidArgument("fgm_params: null");
    if (!(p->gradient_weight >= 0.0)) throw InvalidArgument("MlParams: omega must be >= 0");
    if (!(p->regularization > 0.0)) throw InvalidArgument("MlParams: eps_r must be > 0");
    if (p->n_small_iterations < 1 || p->n_big_iterations < 1)
        throw InvalidArgument("MlParams: iteration counts must be >= 1");
    if (p->small_size < 1) throw InvalidArgument("MlParams: low_res_threshold must be >= 1");
    // fp32 representability of the two weights (the only fp32 restriction).
    const float e = float(p->regularization), o = float(p->gradient_weight);
    if (!(e >= 1.17549435e-38f) || !std::isfinite(e) || !std::isfinite(o))
        throw InvalidArgument("MlParams: eps_r / omega not representable in fp32");
}

// level_schedule (multilevel.cpp:17-44): same integer/libm arithmetic.
std::vector<Level> schedule(int W, int H, const fgm_params* p) {
    if (W < 1 || H < 1) throw InvalidArgument("level_schedule: size must be >= 1x1");
    validate(p);
    const unsigned m = unsigned(std::max(W, H));
    int n = m > 1 ? int(std::bit_width(m - 1)) : 0;
    if (n < 1) n = 1;
    std::vector<Level> out;
    out.reserve(size_t(n));
    for (int l = 1; l <= n; ++l) {
        int w, h;
        if (l == n) {
            w = W;
            h = H;
        } else {
            const double e = double(l) / double(n);
            w = int(std::llround(std::pow(double(W), e)));
            h = int(std::llround(std::pow(double(H), e)));
        }
        const int it = std::max(w, h) <= p->small_size ? p->n_small_iterations : p->n_big_iterations;
        out.push_back({w, h, it});
    }
    return out;
}

// Split `iters` sweeps into fused passes with a compiled K.
std::vector<int> passes_for(int iters) {
    static const int ks[] = {4, 3, 2, 1};
    std::vector<int> out;
    while (iters > 0) {
        for (int k : ks)
            if (k <= iters) {
                out.push_back(k);
                iters -= k;
                break;
            }
    }
    return out;
}

// ---- profiling -------------------------------------------------------------
struct ProfRec {
    cudaEvent_t a, b;
    int which;
    double bytes;
};
std::mutex g_prof_mu;
bool g_prof_on = false;
std::vector<ProfRec> g_prof;
long long g_launches[4] = {0, 0, 0, 0};  // sweep, resample (I/alpha pyramid), coarse, upsample (F/B)
double g_ms[4] = {0, 0, 0, 0}, g_bytes[4] = {0, 0, 0, 0};

// Events come from a free list (created once, reused after each drain) so
// that profiling adds no host-side event creation to the timed launches.
std::vector<cudaEvent_t> g_ev_free;

cudaEvent_t prof_event() {  // caller holds g_prof_mu
    if (!g_ev_free.empty()) {
        cudaEvent_t e = g_ev_free.back();
        g_ev_free.pop_back();
        return e;
    }
    cudaEvent_t e;
    ck(cudaEventCreate(&e), "cudaEventCreate");
    return e;
}

struct ProfScope {
    cudaEvent_t a = nullptr, b = nullptr;
    cudaStream_t s;
    int which;
    double bytes;
    ProfScope(cudaStream_t s_, int which_, double bytes_) : s(s_), which(which_), bytes(bytes_) {
        {
            std::lock_guard<std::mutex> g(g_prof_mu);
            if (!g_prof_on) return;
            a = prof_event();
            b = prof_event();
        }
        ck(cudaEventRecord(a, s), "cudaEventRecord");
    }
    ~ProfScope() {
        if (!a) return;
        cudaEventRecord(b, s);
        std::lock_guard<std::mutex> g(g_prof_mu);
        g_prof.push_back({a, b, which, bytes});
    }
};

// Timeline of the last drained launches (kind, start, end in ms from the
// first recorded launch), for fgm_profile_timeline.
struct TimeRec {
    int which;
    double t0, t1;
};
std::vector<TimeRec> g_timeline;

void prof_drain() {
    std::lock_guard<std::mutex> g(g_prof_mu);
    if (!g_prof.empty()) g_timeline.clear();
    for (auto& r : g_prof) {
        cudaEventSynchronize(r.b);
        float ms = 0, t0 = 0, t1 = 0;
        cudaEventElapsedTime(&ms, r.a, r.b);
        cudaEventElapsedTime(&t0, g_prof.front().a, r.a);
        cudaEventElapsedTime(&t1, g_prof.front().a, r.b);
        g_timeline.push_back({r.which, t0, t1});
        g_launches[r.which] += 1;
        g_ms[r.which] += ms;
        g_bytes[r.which] += r.bytes;
    }
    for (auto& r : g_prof) {
        g_ev_free.push_back(r.a);
        g_ev_free.push_back(r.b);
    }
    g_prof.clear();
}

// ---- device checks ----------------------------------------------------------
void require_device() {
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess || n == 0)
        throw RuntimeError(std::string("no CUDA device available (") + cudaGetErrorString(e) +
                           "); fgmatte_b200 has no CPU fallback");
}

// The library's own stream-ordered memory pool on the current device.  Its
// release threshold is unbounded: a solve's workspace (tens of GB for a large
// batch) stays mapped for the next call instead of being unmapped and mapped
// again at every synchronisation; fgm_release_memory() returns it.  The
// process's default pool (used by other libraries) is left untouched.
cudaMemPool_t device_pool() {
    static PerDevice<cudaMemPool_t> pools;
    cudaMemPool_t p = nullptr;
    ck(pools.get(p, [](int dev, cudaMemPool_t& v) {
           cudaMemPoolProps props{};
           props.allocType = cudaMemAllocationTypePinned;
           props.handleTypes = cudaMemHandleTypeNone;
           props.location.type = cudaMemLocationTypeDevice;
           props.location.id = dev;
           cudaError_t e = cudaMemPoolCreate(&v, &props);
           if (e != cudaSuccess) return e;
           unsigned long long thr = ~0ull;
           return cudaMemPoolSetAttribute(v, cudaMemPoolAttrReleaseThreshold, &thr);
       }),
       "cudaMemPoolCreate");
    return p;
}

template <class T>
void pool_alloc(T** p, size_t bytes, cudaStream_t s, const char* what) {
    ck(cudaMallocFromPoolAsync(reinterpret_cast<void**>(p), bytes, device_pool(), s), what);
}

ResampleJob rjob(const float* src, float* dst, int sw, int sh, int dw, int dh, int np, int spitch, int dpitch) {
    ResampleJob r{};
    r.src = src;
    r.dst = dst;
    r.sw = sw;
    r.sh = sh;
    r.dw = dw;
    r.dh = dh;
    r.nplanes = np;
    r.spitch = spitch;
    r.dpitch = dpitch;
    r.spstride = (long long)spitch * sh;
    r.dpstride = (long long)dpitch * dh;
    r.sx = double(sw) / double(dw);  // make_taps' scale, image.cpp:73
    r.sy = double(sh) / double(dh);
    r.idx32 = (long long)np * std::max(r.spstride, r.dpstride) < (1ll << 31) ? 1 : 0;
    return r;
}

// 16-byte cp.async needs every row start 16-byte aligned.
int vec4_ok(const SweepJob& j) {
    auto al16 = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
    return (j.ipitch % 4 == 0) && (j.fpitch % 4 == 0) && (j.istride % 4 == 0) && (j.fstride % 4 == 0) &&
                   al16(j.img) && al16(j.alpha) && al16(j.fg_in) && al16(j.bg_in)
               ? 1
               : 0;
}

// ---- stream-ordered workspace ----------------------------------------------
// Debug guard mode (fgm_set_debug_guards): every carved region is followed by
// a guard of kGuardBytes filled with a byte pattern; check_guards() (called at
// the end of a solve, synchronously) fails the call if a kernel wrote past a
// region (level buffers, pass ping-pong, boundary streams, job descriptors).
std::atomic<int> g_debug_guards{0};
constexpr size_t kGuardBytes = 4096;
constexpr unsigned char kGuardByte = 0xA5;

struct Arena {
    char* base = nullptr;
    size_t size = 0, off = 0;
    cudaStream_t s = nullptr;
    std::vector<char*> guards;
    bool guarded_ = false;  // guard mode latched at reserve()
    void reserve(size_t bytes, cudaStream_t st, size_t max_takes = 8) {
        s = st;
        guarded_ = g_debug_guards.load() != 0;
        size = bytes + (guarded_ ? max_takes * kGuardBytes : 0);
        if (size) pool_alloc(&base, size, s, "cudaMallocFromPoolAsync");
    }
    template <class T>
    T* take(size_t count) {
        const size_t bytes = (count * sizeof(T) + 255) & ~size_t(255);
        const size_t gb = guarded_ ? kGuardBytes : 0;
        if (off + bytes + gb > size) throw RuntimeError("internal: arena overflow");
        T* p = reinterpret_cast<T*>(base + off);
        off += bytes;
        if (gb) {
            guards.push_back(base + off);
            ck(cudaMemsetAsync(base + off, kGuardByte, gb, s), "cudaMemsetAsync(guard)");
            off += gb;
        }
        return p;
    }
    void check_guards(cudaStream_t st) {
        if (guards.empty()) return;
        std::vector<unsigned char> h(kGuardBytes);
        ck(cudaStreamSynchronize(st), "cudaStreamSynchronize(guards)");
        for (size_t i = 0; i < guards.size(); ++i) {
            ck(cudaMemcpy(h.data(), guards[i], kGuardBytes, cudaMemcpyDeviceToHost), "cudaMemcpy(guard)");
            for (unsigned char c : h)
                if (c != kGuardByte)
                    throw RuntimeError("debug guard: workspace region " + std::to_string(i) + " was overrun");
        }
    }
    ~Arena() {
        if (base) cudaFreeAsync(base, s);
    }
};

inline size_t al(size_t bytes) { return (bytes + 255) & ~size_t(255); }

// ---- the batched multi-level solve ----------------------------------------
struct ImageIO {
    const float* img;
    const float* alpha;
    int W, H;
    float* fg;
    float* bg;
    float* const* level_fg;  // optional per-level dumps (n levels)
    float* const* level_bg;
    // fp64 host path (fgm_ml_solve_host_f64): the caller's fp64 input on the
    // device (the coarse kernel reads it instead of img / alpha) and, for an
    // image whose every level is coarse, fp64 outputs written by that kernel
    const double* img64 = nullptr;
    const double* alpha64 = nullptr;
    double* fg64 = nullptr;
    double* bg64 = nullptr;
};

// Levels handled by the coarse kernel (K4): the schedule's leading levels of
// at most kCoarseCap pixels.
int coarse_levels(const std::vector<Level>& lv) {
    int nc = 0;
    while (nc < int(lv.size()) && nc < kMaxCoarseLevels &&
           size_t(lv[size_t(nc)].w) * lv[size_t(nc)].h <= size_t(kCoarseCap))
        ++nc;
    return nc;
}

struct Plan {
    ImageIO io;
    std::vector<Level> lv;
    int nc = 0;                      // number of coarse levels (K4)
    size_t max_sub = 0;              // max pixels over levels < n-1
    size_t max_lvl = 0;              // max pixels over all levels
    std::vector<size_t> ia_off;      // per level: float offset of its I/alpha block in lvlIA
    size_t ia_floats = 0;            // all big sub-top levels' I/alpha (4 pitched planes each)
    bool multipass = false;
    size_t stream_floats = 0;        // per pass, max over big levels
    int max_bands = 0;
    // carved workspace
    float *lvlIA = nullptr, *fbInit = nullptr, *fbTmp = nullptr, *fbOut = nullptr, *stream = nullptr;
};

void plan_image(Plan& P, const fgm_params* p) {
    P.lv = schedule(P.io.W, P.io.H, p);
    const int n = int(P.lv.size());
    P.nc = coarse_levels(P.lv);
    if (P.nc == 0) throw RuntimeError("internal: first level exceeds the coarse capacity");
    P.ia_off.assign(size_t(n), 0);
    for (int l = 0; l < n; ++l) {
        const size_t px = size_t(level_pitch(P.lv[size_t(l)].w)) * P.lv[size_t(l)].h;
        P.max_lvl = std::max(P.max_lvl, px);
        if (l < n - 1) P.max_sub = std::max(P.max_sub, px);
        if (l >= P.nc && l < n - 1) {  // every level's I/alpha is resampled up front
            P.ia_off[size_t(l)] = P.ia_floats;
            P.ia_floats += (4 * px + 63) / 64 * 64;
        }
        if (l >= P.nc) {
            for (int K : passes_for(P.lv[size_t(l)].iters)) {
                // (sized for the latency kernel's shorter bands: the larger count)
                P.stream_floats = std::max(P.stream_floats, sweep_stream_floats(P.lv[size_t(l)].w, P.lv[size_t(l)].h, K,
                                                                                kLatBandRows));
                P.max_bands = std::max(P.max_bands, sweep_bands(P.lv[size_t(l)].h, K, kLatBandRows));
            }
            if (passes_for(P.lv[size_t(l)].iters).size() > 1) P.multipass = true;
        }
    }
}

size_t plan_bytes(const Plan& P) {
    if (P.nc == int(P.lv.size())) return 0;
    size_t b = 0;
    b += al(std::max<size_t>(P.ia_floats, 1) * sizeof(float));   // lvlIA (all levels)
    b += al(6 * P.max_lvl * sizeof(float));                       // fbInit
    if (P.multipass) b += al(6 * P.max_lvl * sizeof(float));      // fbTmp
    b += al(6 * std::max<size_t>(P.max_sub, 1) * sizeof(float));  // fbOut
    b += al(P.stream_floats * sizeof(float));
    return b;
}

void carve(Plan& P, Arena& A) {
    if (P.nc == int(P.lv.size())) return;
    P.lvlIA = A.take<float>(std::max<size_t>(P.ia_floats, 1));
    P.fbInit = A.take<float>(6 * P.max_lvl);
    if (P.multipass) P.fbTmp = A.take<float>(6 * P.max_lvl);
    P.fbOut = A.take<float>(6 * std::max<size_t>(P.max_sub, 1));
    P.stream = A.take<float>(P.stream_floats);
}

// Pinned staging for job-descriptor uploads: a small per-thread ring, each
// slot reused only after its previous copy completed (an H2D copy from
// pageable memory may synchronise with the stream, which would serialise the
// overlapped host-buffer batch path).
struct PinnedSlot {
    void* p = nullptr;
    size_t cap = 0;
    cudaEvent_t ev = nullptr;
};
struct PinnedRing {
    PinnedSlot slot[4];
    int next = 0;
    ~PinnedRing() {
        for (auto& s : slot) {
            if (s.ev) cudaEventDestroy(s.ev);
            if (s.p) cudaFreeHost(s.p);
        }
    }
    void* stage(const void* src, size_t bytes, cudaStream_t s, void* dst) {
        PinnedSlot& sl = slot[next];
        next = (next + 1) % 4;
        if (sl.ev) ck(cudaEventSynchronize(sl.ev), "cudaEventSynchronize");
        else ck(cudaEventCreateWithFlags(&sl.ev, cudaEventDisableTiming), "cudaEventCreate");
        if (sl.cap < bytes) {
            if (sl.p) cudaFreeHost(sl.p);
            sl.cap = std::max<size_t>(bytes, 1 << 16);
            ck(cudaHostAlloc(&sl.p, sl.cap, cudaHostAllocDefault), "cudaHostAlloc");
        }
        std::memcpy(sl.p, src, bytes);
        ck(cudaMemcpyAsync(dst, sl.p, bytes, cudaMemcpyHostToDevice, s), "cudaMemcpyAsync(jobs)");
        ck(cudaEventRecord(sl.ev, s), "cudaEventRecord");
        return dst;
    }
};
thread_local PinnedRing g_pinned;

// Host-side staging of every job descriptor of one solve: one H2D copy and
// one memset of the dependency counters per solve.
struct JobStage {
    std::vector<unsigned char> host;
    size_t counters = 0;
    template <class T>
    size_t push(const std::vector<T>& v) {
        const size_t off = al(host.size());
        host.resize(off + v.size() * sizeof(T));
        std::memcpy(host.data() + off, v.data(), v.size() * sizeof(T));
        return off;
    }
};

// Ticket order of a sweep launch: band-major across its jobs, so that the
// bands running at any moment belong to many images (no pipeline fill per
// image) and every band's predecessor has a smaller ticket.
// Ticket order of a launch's bands: critical path first.  Band q of image i
// can start ~q*lag steps after the image's band 0 (the boundary-stream lag of
// 32 rows + a 16-column chunk) and the image's chain ends (nb-1)*lag + w steps
// after that, so images get a start offset S_i = -((nb_i-1)*lag + w_i) and
// tickets follow S_i + q*lag.  Within an image the order is q ascending (an
// awaited band always holds an earlier ticket: no deadlock); the tall/wide
// images' long chains start first instead of forming the launch's tail.
std::vector<int2> band_order(const std::vector<SweepJob>& sj, int rows) {
    const double lag = rows + kChunk;
    struct Key {
        double k;
        int i, q;
    };
    std::vector<Key> keys;
    for (size_t i = 0; i < sj.size(); ++i) {
        const double S = -((sj[i].nb - 1) * lag + sj[i].w);
        for (int q = 0; q < sj[i].nb; ++q) keys.push_back({S + q * lag, int(i), q});
    }
    std::stable_sort(keys.begin(), keys.end(), [](const Key& a, const Key& b) { return a.k < b.k; });
    std::vector<int2> ord;
    ord.reserve(keys.size() * 3);
    for (const Key& k : keys)
        for (int c = 0; c < 3; ++c) ord.push_back(make_int2(k.i, 3 * k.q + c));
    return ord;
}

// 1: fused I/alpha pyramid (pyramid_kernel), 0 (default): one resample launch
// per level; the fused pass measured slower
std::atomic<int> g_pyramid_mode{0};

// Persistent per-device count of timed-out boundary-stream waits (sweep.cu).
int* device_fault_counter() {
    static PerDevice<int*> ctr;
    int* p = nullptr;
    ck(ctr.get(p, [](int, int*& v) {
           cudaError_t e = cudaMalloc(reinterpret_cast<void**>(&v), sizeof(int));
           return e == cudaSuccess ? cudaMemset(v, 0, sizeof(int)) : e;
       }),
       "cudaMalloc(fault counter)");
    return p;
}

int read_faults() {
    int v = 0;
    ck(cudaMemcpy(&v, device_fault_counter(), sizeof(int), cudaMemcpyDeviceToHost), "cudaMemcpy(fault counter)");
    return v;
}

// ticket[0]: the launch's band ticket, ticket[1]: its abort flag (both zeroed)
// lat: the jobs are cut into kLatBandRows-row bands for the latency kernel
cudaError_t launch_sweep_passes(int K, const SweepJob* jd, const int2* od, int bands, unsigned* ticket, float eps,
                                float omega, bool lat, cudaStream_t s) {
    return (lat ? launch_sweep_ws : launch_sweep)(K, jd, od, 3 * bands, ticket, eps, omega,
                                                  reinterpret_cast<int*>(ticket + 1), device_fault_counter(), s);
}

enum LaunchKind { kCoarse, kResample, kUpsample, kSweep, kCopy, kPyramid };
struct LaunchRec {
    LaunchKind kind;
    int K, njobs, total_bands;
    size_t job_off, ticket, order_off;
    long long max_rows;
    double bytes;
    void* dst = nullptr;
    const void* src = nullptr;
    int side = 0;   // 1: runs on the side stream, then records event `ev`
    int ev = -1;    // side: event to record after; main: event to wait for before
    int lat = 0;    // kSweep: latency kernel (kLatBandRows-row bands)
};

// The side stream of the calling thread's device (I/alpha pyramid, which
// depends only on the inputs and overlaps the main stream's coarse levels,
// upsamples and sweeps), and a pool of events.
struct SideStream {
    int dev = -1;
    cudaStream_t s = nullptr;
    std::vector<cudaEvent_t> ev;
    cudaEvent_t event(size_t i) {
        while (ev.size() <= i) {
            cudaEvent_t e;
            ck(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "cudaEventCreate");
            ev.push_back(e);
        }
        return ev[i];
    }
};
thread_local SideStream g_side;
// persistent blocks per SM of the side-stream pyramid launches (16 fills the GPU)
constexpr int kSideBlocksPerSm = 16;

SideStream& side_stream() {
    int dev = 0;
    ck(cudaGetDevice(&dev), "cudaGetDevice");
    if (g_side.dev != dev) {  // (a thread that switches devices re-creates it; the old one leaks)
        g_side = SideStream{};
        int lo = 0, hi = 0;  // lowest priority: its blocks yield SM slots to the main stream's
        ck(cudaDeviceGetStreamPriorityRange(&lo, &hi), "cudaDeviceGetStreamPriorityRange");
        ck(cudaStreamCreateWithPriority(&g_side.s, cudaStreamNonBlocking, lo), "cudaStreamCreate");
        g_side.dev = dev;
    }
    return g_side;
}

void solve_batch(std::vector<ImageIO>& ios, const fgm_params* p, cudaStream_t s) {
    validate(p);
    require_device();
    const float eps = float(p->regularization), omega = float(p->gradient_weight);
    const double eps64 = p->regularization, omega64 = p->gradient_weight;  // the coarse kernel is fp64
    std::vector<Plan> plans(ios.size());
    for (size_t i = 0; i < ios.size(); ++i) {
        if (!ios[i].img || !ios[i].alpha || !ios[i].fg || !ios[i].bg) throw InvalidArgument("null buffer");
        plans[i].io = ios[i];
        plan_image(plans[i], p);
    }
    size_t ws = 0;
    int J = 0;
    for (auto& P : plans) {
        ws += plan_bytes(P);
        J = std::max(J, int(P.lv.size()) - P.nc);
    }
    Arena W;
    W.reserve(ws, s, 5 * plans.size() + 1);
    for (auto& P : plans) carve(P, W);

    JobStage st;
    std::vector<LaunchRec> launches;

    // ---- K4: every image's coarse prefix ---------------------------------
    {
        std::vector<CoarseJob> cj(plans.size());
        double bytes = 0;
        for (size_t i = 0; i < plans.size(); ++i) {
            const Plan& P = plans[i];
            CoarseJob& c = cj[i];
            std::memset(&c, 0, sizeof(c));
            c.img = P.io.img;
            c.alpha = P.io.alpha;
            c.img64 = P.io.img64;
            c.alpha64 = P.io.alpha64;
            c.W = P.io.W;
            c.H = P.io.H;
            c.nlev = P.nc;
            for (int l = 0; l < P.nc; ++l) {
                c.lw[l] = P.lv[size_t(l)].w;
                c.lh[l] = P.lv[size_t(l)].h;
                c.lit[l] = P.lv[size_t(l)].iters;
                if (P.io.level_fg) {
                    c.lvl_fg[l] = P.io.level_fg[l];
                    c.lvl_bg[l] = P.io.level_bg[l];
                }
            }
            const Level Lc = P.lv[size_t(P.nc - 1)];
            const size_t n = size_t(Lc.w) * Lc.h;
            if (P.nc == int(P.lv.size())) {
                c.fg_out = P.io.fg;
                c.bg_out = P.io.bg;
                c.fg_out64 = P.io.fg64;
                c.bg_out64 = P.io.bg64;
                c.out_pitch = Lc.w;
            } else {
                c.out_pitch = level_pitch(Lc.w);
                c.fg_out = P.fbOut;
                c.bg_out = P.fbOut + 3 * size_t(c.out_pitch) * Lc.h;
            }
            c.out_pstride = (long long)c.out_pitch * Lc.h;
            bytes += 24.0 * double(n);
        }
        launches.push_back({kCoarse, 0, int(cj.size()), 0, st.push(cj), 0, 0, 0, bytes});
    }

    // ---- I/alpha pyramid of every big sub-top level, on the side stream ----
    // Fused (default): one pass over each full-res input emits every level
    // (pyramid_kernel); its event (index J + 3) gates the first sweep of
    // every sub-top level.  Per level (FGM_PYRAMID=0): step j's resample
    // launch records event j and step j's sweep waits for it.
    const bool fused_pyr = g_pyramid_mode.load() != 0;
    bool pyr_fits = true;
    for (const auto& P : plans) pyr_fits = pyr_fits && int(P.lv.size()) - 1 - P.nc <= kMaxPyr;
    const int pyr_ev = J + 3;
    bool pyr_launch = false;
    if (fused_pyr && pyr_fits) {
        std::vector<PyrJob> pj;
        long long tiles = 0;
        double bytes = 0;
        for (auto& P : plans) {
            const int n = int(P.lv.size());
            PyrJob q{};
            q.img = P.io.img;
            q.alpha = P.io.alpha;
            q.W = P.io.W;
            q.H = P.io.H;
            for (int l = P.nc; l < n - 1; ++l) {
                const Level L = P.lv[size_t(l)];
                q.lw[q.nlev] = L.w;
                q.lh[q.nlev] = L.h;
                q.pitch[q.nlev] = level_pitch(L.w);
                q.sx[q.nlev] = double(P.io.W) / double(L.w);  // make_taps' scale, image.cpp:73
                q.sy[q.nlev] = double(P.io.H) / double(L.h);
                q.rsx[q.nlev] = 1.0 / q.sx[q.nlev];
                q.rsy[q.nlev] = 1.0 / q.sy[q.nlev];
                q.out[q.nlev] = P.lvlIA + P.ia_off[size_t(l)];
                bytes += 16.0 * double(L.w) * L.h;
                ++q.nlev;
            }
            if (q.nlev == 0) continue;
            q.tcols = (q.W + kPyrTW - 1) / kPyrTW;
            q.tile_base = int(tiles);
            tiles += pyramid_tiles(q.W, q.H);
            bytes += 16.0 * double(q.W) * q.H * (1.0 + 1.0 / kPyrTH);
            pj.push_back(q);
        }
        if (!pj.empty()) {
            LaunchRec lr{kPyramid, 0, int(pj.size()), 0, st.push(pj), 0, 0, tiles, bytes};
            lr.side = 1;
            lr.ev = pyr_ev;
            launches.push_back(lr);
            pyr_launch = true;
        }
    }
    for (int j = 0; j < J && !pyr_launch; ++j) {
        std::vector<ResampleJob> rj;
        long long tiles = 0;
        double rbytes = 0;
        for (auto& P : plans) {
            const int n = int(P.lv.size());
            const int l = n - J + j;
            if (l < P.nc || l >= n - 1) continue;
            const Level L = P.lv[size_t(l)];
            const long long px = (long long)L.w * L.h, fpx = (long long)P.io.W * P.io.H;
            const int pp = level_pitch(L.w);
            const long long pps = (long long)pp * L.h;
            float* ia = P.lvlIA + P.ia_off[size_t(l)];
            rj.push_back(rjob(P.io.img, ia, P.io.W, P.io.H, L.w, L.h, 3, P.io.W, pp));
            rj.push_back(rjob(P.io.alpha, ia + 3 * pps, P.io.W, P.io.H, L.w, L.h, 1, P.io.W, pp));
            rbytes += 4.0 * 4 * (double(px) + std::min<double>(double(fpx), 4.0 * px));
        }
        if (rj.empty()) continue;
        for (auto& r : rj) {
            r.tile_base = int(tiles);
            tiles += resample_tiles(r.dw, r.dh);
        }
        LaunchRec lr{kResample, 0, int(rj.size()), 0, st.push(rj), 0, 0, tiles, rbytes};
        lr.side = 1;
        lr.ev = j;
        launches.push_back(lr);
    }
    std::vector<char> has_ia(size_t(J), 0);
    for (const auto& r : launches)
        if (r.side && r.kind == kResample) has_ia[size_t(r.ev)] = 1;

    // ---- big levels, aligned so that every image's top level is step J-1 --
    for (int j = 0; j < J; ++j) {
        std::vector<ResampleJob> rj, uj;  // resample (I/alpha) and upsample (F/B) jobs
        long long max_rows = 0;
        double rbytes = 0, ubytes = 0;
        struct Active {
            Plan* P;
            int l;
        };
        std::vector<Active> act;
        for (auto& P : plans) {
            const int n = int(P.lv.size());
            const int l = n - J + j;
            if (l < P.nc) continue;
            act.push_back({&P, l});
            const Level L = P.lv[size_t(l)], Lp = P.lv[size_t(l - 1)];
            const long long px = (long long)L.w * L.h, ppx = (long long)Lp.w * Lp.h;
            const int pp = level_pitch(L.w);
            // the previous level's output: the coarse kernel's or a sweep's (both
            // pitched); levels grow, so this is an upsample (staged kernel)
            const ResampleJob fj = rjob(P.fbOut, P.fbInit, Lp.w, Lp.h, L.w, L.h, 6, level_pitch(Lp.w), pp);
            if (upsample_ok(Lp.w, Lp.h, L.w, L.h)) {
                uj.push_back(fj);
                ubytes += 4.0 * 6 * (double(px) + double(ppx));
            } else {
                rj.push_back(fj);
                rbytes += 4.0 * 6 * (double(px) + double(ppx));
            }

        }
        if (act.empty()) continue;
        for (auto& r : rj) {
            r.tile_base = int(max_rows);
            max_rows += resample_tiles(r.dw, r.dh);
        }
        if (!rj.empty()) launches.push_back({kResample, 0, int(rj.size()), 0, st.push(rj), 0, 0, max_rows, rbytes});
        long long up_tiles = 0;
        for (auto& r : uj) {
            r.tile_base = int(up_tiles);
            up_tiles += upsample_tiles(r.dw, r.dh);
        }
        if (!uj.empty()) launches.push_back({kUpsample, 0, int(uj.size()), 0, st.push(uj), 0, 0, up_tiles, ubytes});
        size_t max_passes = 0;
        for (auto& a : act) max_passes = std::max(max_passes, passes_for(a.P->lv[size_t(a.l)].iters).size());
        for (size_t pi = 0; pi < max_passes; ++pi) {
            for (int K : {4, 3, 2, 1}) {
                std::vector<SweepJob> sj;
                int total = 0;
                double sbytes = 0;
                size_t max_stream = 0;
                const size_t ticket = st.counters;
                st.counters += 2;  // ticket, abort flag
                int njobs = 0;
                for (auto& a : act) {
                    const std::vector<int> ps = passes_for(a.P->lv[size_t(a.l)].iters);
                    njobs += pi < ps.size() && ps[pi] == K ? 1 : 0;
                }
                // a few images: the wavefront chain bounds the launch (latency kernel)
                const bool lat = njobs <= kLatMaxJobs;
                const int rows = lat ? kLatBandRows : kBandRows;
                for (auto& a : act) {
                    Plan& P = *a.P;
                    const std::vector<int> ps = passes_for(P.lv[size_t(a.l)].iters);
                    if (pi >= ps.size() || ps[pi] != K) continue;
                    const Level L = P.lv[size_t(a.l)];
                    const int n = int(P.lv.size());
                    const long long px = (long long)L.w * L.h;
                    const int pp = level_pitch(L.w);
                    const long long pps = (long long)pp * L.h;
                    const bool last = pi + 1 == ps.size();
                    const bool top = a.l == n - 1;
                    float* bufs[2] = {P.fbTmp, P.fbInit};  // pass ping-pong (pitched)
                    const float* in = pi == 0 ? P.fbInit : bufs[(pi - 1) & 1];
                    SweepJob J1{};
                    // the top level reads/writes the caller's dense planes, the
                    // others the solver's pitched level buffers
                    float* ia = P.lvlIA + P.ia_off[size_t(a.l)];
                    J1.img = top ? P.io.img : ia;
                    J1.alpha = top ? P.io.alpha : ia + 3 * pps;
                    J1.ipitch = top ? L.w : pp;
                    J1.istride = top ? px : pps;
                    J1.fg_in = in;
                    J1.bg_in = in + 3 * pps;
                    J1.fpitch = pp;
                    J1.fstride = pps;
                    const bool user_out = last && top;
                    if (last) {
                        J1.fg_out = top ? P.io.fg : P.fbOut;
                        J1.bg_out = top ? P.io.bg : P.fbOut + 3 * pps;
                    } else {
                        J1.fg_out = bufs[pi & 1];
                        J1.bg_out = bufs[pi & 1] + 3 * pps;
                    }
                    J1.opitch = user_out ? L.w : pp;
                    J1.ostride = user_out ? px : pps;
                    J1.stream = P.stream;
                    J1.w = L.w;
                    J1.h = L.h;
                    J1.nb = sweep_bands(L.h, K, rows);
                    J1.band_base = total;
                    J1.vec4 = vec4_ok(J1);
                    total += J1.nb;
                    max_stream = std::max(max_stream, sweep_stream_floats(L.w, L.h, K, rows));
                    sbytes += 64.0 * double(px);
                    sj.push_back(J1);
                }
                if (sj.empty()) {
                    st.counters -= 2;
                    continue;
                }
                const size_t off = st.push(sj);
                const size_t ooff = st.push(band_order(sj, rows));
                LaunchRec lr{kSweep, K, int(sj.size()), total, off, ticket, ooff, (long long)max_stream, sbytes};
                lr.lat = lat ? 1 : 0;
                if (pi == 0 && has_ia[size_t(j)]) lr.ev = j;  // this step's I/alpha pyramid level
                if (pi == 0 && pyr_launch && j < J - 1) lr.ev = pyr_ev;
                launches.push_back(lr);
            }
        }
        for (auto& a : act) {  // per-level dumps (debug API)
            Plan& P = *a.P;
            if (!P.io.level_fg) continue;
            const Level L = P.lv[size_t(a.l)];
            const bool top = a.l == int(P.lv.size()) - 1;
            const int sp = top ? L.w : level_pitch(L.w);
            const float* f = top ? P.io.fg : P.fbOut;
            const float* b = top ? P.io.bg : P.fbOut + 3 * size_t(sp) * L.h;
            // 3 planes = 3h rows of the source pitch (plane stride = pitch * h)
            if (P.io.level_fg[a.l])
                launches.push_back({kCopy, 0, L.w, 3 * L.h, 0, 0, 0, sp, 0.0, P.io.level_fg[a.l], f});
            if (P.io.level_bg[a.l])
                launches.push_back({kCopy, 0, L.w, 3 * L.h, 0, 0, 0, sp, 0.0, P.io.level_bg[a.l], b});
        }
    }

    Arena B;
    B.reserve(al(st.host.size()) + al(std::max<size_t>(st.counters, 1) * sizeof(unsigned)), s, 2);
    unsigned char* djobs = B.take<unsigned char>(st.host.size());
    unsigned* dctr = B.take<unsigned>(std::max<size_t>(st.counters, 1));
    ck(cudaMemsetAsync(dctr, 0, std::max<size_t>(st.counters, 1) * sizeof(unsigned), s), "cudaMemsetAsync");
    g_pinned.stage(st.host.data(), st.host.size(), s, djobs);

    // the side stream starts after everything enqueued on s so far (inputs,
    // job uploads) and s waits for all of its work at the end -- also when a
    // launch below throws: the join is a scope guard declared after the
    // arenas, so it runs before their stream-ordered frees
    SideStream& side = side_stream();
    const cudaEvent_t ev_start = side.event(size_t(J)), ev_end = side.event(size_t(J) + 1);
    bool any_side = false;
    for (const LaunchRec& r : launches) any_side = any_side || r.side;
    struct SideJoin {
        bool armed = false;
        cudaStream_t side, caller;
        cudaEvent_t ev;
        ~SideJoin() {
            if (!armed) return;
            cudaEventRecord(ev, side);
            cudaStreamWaitEvent(caller, ev, 0);
        }
    } join{false, side.s, s, ev_end};
    if (any_side) {
        ck(cudaEventRecord(ev_start, s), "cudaEventRecord");
        ck(cudaStreamWaitEvent(side.s, ev_start, 0), "cudaStreamWaitEvent");
        join.armed = true;
    }

    for (const LaunchRec& r : launches) {
        if (r.side && r.kind == kPyramid) {  // the whole I/alpha pyramid
            ProfScope ps(side.s, 1, r.bytes);
            ck(launch_pyramid(reinterpret_cast<const PyrJob*>(djobs + r.job_off), r.njobs, r.max_rows, side.s),
               "pyramid_kernel");
            ck(cudaEventRecord(side.event(size_t(r.ev)), side.s), "cudaEventRecord");
            continue;
        }
        if (r.side) {  // I/alpha pyramid level
            ProfScope ps(side.s, 1, r.bytes);
            ck(launch_resample(reinterpret_cast<const ResampleJob*>(djobs + r.job_off), r.njobs, r.max_rows, side.s,
                               kSideBlocksPerSm),
               "resample_kernel");
            ck(cudaEventRecord(side.event(size_t(r.ev)), side.s), "cudaEventRecord");
            continue;
        }
        if (r.ev >= 0) ck(cudaStreamWaitEvent(s, side.event(size_t(r.ev)), 0), "cudaStreamWaitEvent");
        switch (r.kind) {
            case kPyramid: break;  // (side stream only)
            case kCoarse: {
                ProfScope ps(s, 2, r.bytes);
                ck(launch_coarse(reinterpret_cast<const CoarseJob*>(djobs + r.job_off), r.njobs, eps64, omega64, s),
                   "coarse_kernel");
                break;
            }
            case kResample: {
                ProfScope ps(s, 1, r.bytes);
                ck(launch_resample(reinterpret_cast<const ResampleJob*>(djobs + r.job_off), r.njobs, r.max_rows, s),
                   "resample_kernel");
                break;
            }
            case kUpsample: {
                ProfScope ps(s, 3, r.bytes);
                ck(launch_upsample(reinterpret_cast<const ResampleJob*>(djobs + r.job_off), r.njobs, r.max_rows, s),
                   "upsample_kernel");
                break;
            }
            case kSweep: {
                ck(launch_stream_fill(reinterpret_cast<const SweepJob*>(djobs + r.job_off), r.njobs, r.K,
                                      size_t(r.max_rows), s),
                   "stream_fill_kernel");
                ProfScope ps(s, 0, r.bytes);
                const SweepJob* jd = reinterpret_cast<const SweepJob*>(djobs + r.job_off);
                const int2* od = reinterpret_cast<const int2*>(djobs + r.order_off);
                ck(launch_sweep_passes(r.K, jd, od, r.total_bands, dctr + r.ticket, eps, omega, r.lat != 0, s),
                   "sweep_kernel");
                break;
            }
            case kCopy:  // njobs = width, total_bands = rows, max_rows = source pitch (floats)
                ck(cudaMemcpy2DAsync(r.dst, size_t(r.njobs) * sizeof(float), r.src, size_t(r.max_rows) * sizeof(float),
                                     size_t(r.njobs) * sizeof(float), size_t(r.total_bands), cudaMemcpyDeviceToDevice, s),
                   "cudaMemcpy2DAsync");
                break;
        }
    }
    if (any_side) {  // nothing of this call stays outstanding on the side stream
        join.armed = false;
        ck(cudaEventRecord(ev_end, side.s), "cudaEventRecord");
        ck(cudaStreamWaitEvent(s, ev_end, 0), "cudaStreamWaitEvent");
    }
    if (W.guarded_ || B.guarded_) {
        W.check_guards(s);
        B.check_guards(s);
    }
}

template <class F>
int guarded(F&& fn) {
    try {
        fn();
        return FGM_OK;
    } catch (const InvalidArgument& e) {
        g_err = e.what();
        return FGM_INVALID_ARGUMENT;
    } catch (const std::exception& e) {
        g_err = e.what();
        return FGM_RUNTIME_ERROR;
    }
}

// A boundary-stream wait that timed out (a band whose predecessor never
// published) aborts its launch; synchronous entry points report it.
void check_faults(int before) {
    if (read_faults() != before)
        throw RuntimeError("sweep: a boundary-stream wait timed out after " +
                           std::to_string(g_spin_timeout_ns.load() / 1000000) +
                           " ms (band hand-over stalled); the launch was aborted and its results are invalid");
}

void check_dims(int w, int h) {
    if (w < 1 || h < 1)
        throw InvalidArgument("Image: dimensions must be >= 1, got " + std::to_string(w) + "x" + std::to_string(h));
}

}  // namespace
}  // namespace fgm

using namespace fgm;

extern "C" {

void fgm_params_default(fgm_params* p) {
    if (!p) return;
    p->regularization = 5e-3;
    p->gradient_weight = 0.1;
    p->n_small_iterations = 10;
    p->n_big_iterations = 2;
    p->small_size = 32;
}

int fgm_params_validate(const fgm_params* p) {
    return guarded([&] { validate(p); });
}

int fgm_level_schedule(int w, int h, const fgm_params* p, int* ow, int* oh, int* oit, int cap) {
    int n = 0;
    const int rc = guarded([&] {
        const auto lv = schedule(w, h, p);
        n = int(lv.size());
        for (int l = 0; l < n && l < cap; ++l) {
            if (ow) ow[l] = lv[size_t(l)].w;
            if (oh) oh[l] = lv[size_t(l)].h;
            if (oit) oit[l] = lv[size_t(l)].iters;
        }
    });
    return rc ? -rc : n;
}

int fgm_ml_solve_f32(const float* image, const float* alpha, int w, int h, const fgm_params* p, float* fg, float* bg,
                     void* stream) {
    return guarded([&] {
        check_dims(w, h);
        std::vector<ImageIO> io{{image, alpha, w, h, fg, bg, nullptr, nullptr}};
        solve_batch(io, p, static_cast<cudaStream_t>(stream));
    });
}

int fgm_ml_solve_levels_f32(const float* image, const float* alpha, int w, int h, const fgm_params* p, float* fg,
                            float* bg, float* const* level_fg, float* const* level_bg, int n_levels, void* stream) {
    return guarded([&] {
        check_dims(w, h);
        const auto lv = schedule(w, h, p);
        if (n_levels != int(lv.size()) || !level_fg || !level_bg)
            throw InvalidArgument("fgm_ml_solve_levels_f32: need one (fg, bg) buffer pair per level (" +
                                  std::to_string(lv.size()) + ")");
        std::vector<ImageIO> io{{image, alpha, w, h, fg, bg, level_fg, level_bg}};
        solve_batch(io, p, static_cast<cudaStream_t>(stream));
    });
}

int fgm_batch_solve_f32(int n_images, const float* const* images, const float* const* alphas, const int* widths,
                        const int* heights, const fgm_params* p, float* const* fgs, float* const* bgs, void* stream) {
    return guarded([&] {
        if (n_images < 0) throw InvalidArgument("fgm_batch_solve_f32: n_images < 0");
        if (n_images == 0) return;
        std::vector<ImageIO> io;
        io.reserve(size_t(n_images));
        for (int i = 0; i < n_images; ++i) {
            check_dims(widths[i], heights[i]);
            io.push_back({images[i], alphas[i], widths[i], heights[i], fgs[i], bgs[i], nullptr, nullptr});
        }
        solve_batch(io, p, static_cast<cudaStream_t>(stream));
    });
}

static int host_solve_impl(const void* image, const void* alpha, int w, int h, const fgm_params* p, void* fg,
                           void* bg, bool f64) {
    return guarded([&] {
        check_dims(w, h);
        validate(p);
        require_device();
        cudaStream_t s;
        ck(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "cudaStreamCreate");
        struct SG {
            cudaStream_t s;
            ~SG() { cudaStreamDestroy(s); }
        } sg{s};
        const size_t n = size_t(w) * h;
        const int faults0 = read_faults();
        Arena A;
        // image + alpha (4 planes) and F + B (6 planes) in fp32; the fp64 path
        // stages the 4 input planes and the 6 output planes in fp64 as well
        A.reserve(al(4 * n * sizeof(float)) + al(6 * n * sizeof(float)) +
                      (f64 ? al(4 * n * sizeof(double)) + al(6 * n * sizeof(double)) : 0),
                  s);
        float* dimg = A.take<float>(4 * n);  // 3 image planes + alpha
        float* dout = A.take<float>(6 * n);
        if (f64) {
            double* staging = A.take<double>(4 * n);
            double* out64 = A.take<double>(6 * n);
            ck(cudaMemcpyAsync(staging, image, 3 * n * sizeof(double), cudaMemcpyHostToDevice, s), "H2D");
            ck(cudaMemcpyAsync(staging + 3 * n, alpha, n * sizeof(double), cudaMemcpyHostToDevice, s), "H2D");
            ck(launch_f64_to_f32(staging, dimg, 4 * n, s), "f64_to_f32");
            // the coarse levels read the fp64 input itself (bitwise the
            // reference's coarse levels); an image that is coarse at every
            // level gets its fp64 result straight from the coarse kernel
            ImageIO one{dimg, dimg + 3 * n, w, h, dout, dout + 3 * n, nullptr, nullptr};
            one.img64 = staging;
            one.alpha64 = staging + 3 * n;
            one.fg64 = out64;
            one.bg64 = out64 + 3 * n;
            std::vector<ImageIO> io{one};
            solve_batch(io, p, s);
            const std::vector<Level> lv = schedule(w, h, p);
            if (coarse_levels(lv) != int(lv.size())) ck(launch_f32_to_f64(dout, out64, 6 * n, s), "f32_to_f64");
            ck(cudaMemcpyAsync(fg, out64, 3 * n * sizeof(double), cudaMemcpyDeviceToHost, s), "D2H");
            ck(cudaMemcpyAsync(bg, out64 + 3 * n, 3 * n * sizeof(double), cudaMemcpyDeviceToHost, s), "D2H");
        } else {
            ck(cudaMemcpyAsync(dimg, image, 3 * n * sizeof(float), cudaMemcpyHostToDevice, s), "H2D");
            ck(cudaMemcpyAsync(dimg + 3 * n, alpha, n * sizeof(float), cudaMemcpyHostToDevice, s), "H2D");
            std::vector<ImageIO> io{{dimg, dimg + 3 * n, w, h, dout, dout + 3 * n, nullptr, nullptr}};
            solve_batch(io, p, s);
            ck(cudaMemcpyAsync(fg, dout, 3 * n * sizeof(float), cudaMemcpyDeviceToHost, s), "D2H");
            ck(cudaMemcpyAsync(bg, dout + 3 * n, 3 * n * sizeof(float), cudaMemcpyDeviceToHost, s), "D2H");
        }
        ck(cudaStreamSynchronize(s), "cudaStreamSynchronize");
        check_faults(faults0);
    });
}

int fgm_batch_solve_host_f32(int n_images, const float* const* images, const float* const* alphas, const int* widths,
                             const int* heights, const fgm_params* p, float* const* fgs, float* const* bgs) {
    return guarded([&] {
        if (n_images < 0) throw InvalidArgument("fgm_batch_solve_host_f32: n_images < 0");
        validate(p);
        for (int i = 0; i < n_images; ++i) check_dims(widths[i], heights[i]);
        if (n_images == 0) return;
        require_device();
        const int faults0 = read_faults();
        // Sub-batches of ~1/64 of the pixels (at least one image each) in
        // kSlots device slots: copy-in runs up to kSlots groups ahead of
        // copy-out, so both PCIe directions stay busy while the (much
        // shorter) solves run in between.  Measured on the C4 batch: 16
        // groups / 4 slots 1812 MP/s, 64 / 8 1965, 128 / 8 1549 (per-group
        // launch overhead).
#ifndef FGM_HOST_GROUPS
#define FGM_HOST_GROUPS 64
#endif
#ifndef FGM_HOST_SLOTS
#define FGM_HOST_SLOTS 8
#endif
        constexpr size_t kGroups = FGM_HOST_GROUPS, kSlots = FGM_HOST_SLOTS;
        size_t total = 0;
        for (int i = 0; i < n_images; ++i) total += size_t(widths[i]) * heights[i];
        const size_t target = std::max<size_t>(total / kGroups, 1);
        std::vector<std::pair<int, int>> groups;  // [begin, end)
        for (int b = 0; b < n_images;) {
            int e = b;
            size_t px = 0;
            while (e < n_images && (e == b || px < target)) px += size_t(widths[e]) * heights[e], ++e;
            groups.push_back({b, e});
            b = e;
        }
        cudaStream_t sc, sin, sout;
        ck(cudaStreamCreateWithFlags(&sc, cudaStreamNonBlocking), "cudaStreamCreate");
        ck(cudaStreamCreateWithFlags(&sin, cudaStreamNonBlocking), "cudaStreamCreate");
        ck(cudaStreamCreateWithFlags(&sout, cudaStreamNonBlocking), "cudaStreamCreate");
        struct SG {
            cudaStream_t a, b, c;
            ~SG() {
                cudaStreamSynchronize(a);
                cudaStreamSynchronize(b);
                cudaStreamSynchronize(c);
                cudaStreamDestroy(a);
                cudaStreamDestroy(b);
                cudaStreamDestroy(c);
            }
        } sg{sc, sin, sout};
        // kSlots device slots of the largest group, 10 floats per pixel each
        size_t gmax = 0;
        for (auto [b, e] : groups) {
            size_t px = 0;
            for (int i = b; i < e; ++i) px += size_t(widths[i]) * heights[i];
            gmax = std::max(gmax, px);
        }
        const size_t slot_floats = 10 * gmax + 64 * size_t(n_images);
        const size_t nslots = std::min(kSlots, groups.size());
        // owned resources, released on every exit (an exception included): the
        // slots once all three streams are idle, then the events
        struct Owned {
            float* dbuf = nullptr;
            std::vector<cudaEvent_t> ev;
            cudaStream_t a, b, c;
            ~Owned() {
                if (dbuf) {
                    cudaStreamSynchronize(a);
                    cudaStreamSynchronize(b);
                    cudaStreamSynchronize(c);
                    cudaFreeAsync(dbuf, c);
                    cudaStreamSynchronize(c);
                }
                for (cudaEvent_t e : ev)
                    if (e) cudaEventDestroy(e);
            }
        } own{nullptr, {}, sin, sout, sc};
        pool_alloc(&own.dbuf, nslots * slot_floats * sizeof(float), sc, "cudaMallocFromPoolAsync");
        float* const dbuf = own.dbuf;
        own.ev.assign(3 * groups.size(), nullptr);
        for (cudaEvent_t& e : own.ev) ck(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "cudaEventCreate");
        cudaEvent_t* const ev_in = own.ev.data();
        cudaEvent_t* const ev_done = ev_in + groups.size();
        cudaEvent_t* const ev_out = ev_done + groups.size();
        ck(cudaStreamSynchronize(sc), "cudaStreamSynchronize");
        for (size_t g = 0; g < groups.size(); ++g) {
            const auto [b, e] = groups[g];
            float* slot = dbuf + (g % nslots) * slot_floats;
            // the slot's previous user (group g - nslots) must have been copied out
            if (g >= nslots) ck(cudaStreamWaitEvent(sin, ev_out[g - nslots], 0), "cudaStreamWaitEvent");
            std::vector<ImageIO> io;
            size_t off = 0;
            for (int i = b; i < e; ++i) {
                const size_t n = size_t(widths[i]) * heights[i];
                float* di = slot + off;
                float* da = di + 3 * n;
                float* dfg = da + n;
                float* dbg = dfg + 3 * n;
                off += (10 * n + 63) / 64 * 64;
                ck(cudaMemcpyAsync(di, images[i], 3 * n * sizeof(float), cudaMemcpyHostToDevice, sin), "H2D");
                ck(cudaMemcpyAsync(da, alphas[i], n * sizeof(float), cudaMemcpyHostToDevice, sin), "H2D");
                io.push_back({di, da, widths[i], heights[i], dfg, dbg, nullptr, nullptr});
            }
            ck(cudaEventRecord(ev_in[g], sin), "cudaEventRecord");
            ck(cudaStreamWaitEvent(sc, ev_in[g], 0), "cudaStreamWaitEvent");
            solve_batch(io, p, sc);
            ck(cudaEventRecord(ev_done[g], sc), "cudaEventRecord");
            ck(cudaStreamWaitEvent(sout, ev_done[g], 0), "cudaStreamWaitEvent");
            for (int i = b; i < e; ++i) {
                const ImageIO& x = io[size_t(i - b)];
                const size_t n = size_t(widths[i]) * heights[i];
                ck(cudaMemcpyAsync(fgs[i], x.fg, 3 * n * sizeof(float), cudaMemcpyDeviceToHost, sout), "D2H");
                ck(cudaMemcpyAsync(bgs[i], x.bg, 3 * n * sizeof(float), cudaMemcpyDeviceToHost, sout), "D2H");
            }
            ck(cudaEventRecord(ev_out[g], sout), "cudaEventRecord");
        }
        ck(cudaStreamSynchronize(sout), "cudaStreamSynchronize");
        ck(cudaStreamSynchronize(sc), "cudaStreamSynchronize");
        check_faults(faults0);
    });
}

int fgm_ml_solve_host_f32(const float* image, const float* alpha, int w, int h, const fgm_params* p, float* fg,
                          float* bg) {
    return host_solve_impl(image, alpha, w, h, p, fg, bg, false);
}

int fgm_ml_solve_host_f64(const double* image, const double* alpha, int w, int h, const fgm_params* p, double* fg,
                          double* bg) {
    return host_solve_impl(image, alpha, w, h, p, fg, bg, true);
}

int fgm_resize_f32(const float* src, int sw, int sh, int nplanes, float* dst, int dw, int dh, void* stream) {
    return guarded([&] {
        if (dw < 1 || dh < 1)
            throw InvalidArgument("resize: target size must be >= 1x1, got " + std::to_string(dw) + "x" +
                                  std::to_string(dh));
        check_dims(sw, sh);
        if (nplanes < 1) throw InvalidArgument("resize: nplanes must be >= 1");
        require_device();
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        Arena A;
        A.reserve(4096, s);
        ResampleJob rj = rjob(src, dst, sw, sh, dw, dh, nplanes, sw, dw);
        rj.tile_base = 0;
        ResampleJob* d = A.take<ResampleJob>(1);
        ck(cudaMemcpyAsync(d, &rj, sizeof(rj), cudaMemcpyHostToDevice, s), "cudaMemcpyAsync(jobs)");
        if (nplanes == 6 && upsample_ok(sw, sh, dw, dh))  // the solver's F/B upsample path
            ck(launch_upsample(d, 1, upsample_tiles(dw, dh), s), "upsample_kernel");
        else
            ck(launch_resample(d, 1, resample_tiles(dw, dh), s), "resample_kernel");
    });
}

int fgm_ml_solve_hwc(const void* image_hwc, const void* alpha, int w, int h, int f64, const fgm_params* p,
                     void* fg_hwc, void* bg_hwc, void* stream) {
    return guarded([&] {
        check_dims(w, h);
        validate(p);
        if (!image_hwc || !alpha || !fg_hwc || !bg_hwc) throw InvalidArgument("ml_foreground_background: null buffer");
        require_device();
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        const size_t n = size_t(w) * h;
        Arena A;
        A.reserve(al(10 * n * sizeof(float)), s);
        float* dimg = A.take<float>(4 * n);  // 3 image planes + alpha
        float* dout = A.take<float>(6 * n);
        ck(launch_hwc_to_planar(image_hwc, f64 != 0, (long long)n, 3, dimg, s), "hwc_to_planar");
        ck(launch_hwc_to_planar(alpha, f64 != 0, (long long)n, 1, dimg + 3 * n, s), "hwc_to_planar");
        std::vector<ImageIO> io{{dimg, dimg + 3 * n, w, h, dout, dout + 3 * n, nullptr, nullptr}};
        solve_batch(io, p, s);
        ck(launch_planar_to_hwc(dout, (long long)n, 3, fg_hwc, f64 != 0, s), "planar_to_hwc");
        ck(launch_planar_to_hwc(dout + 3 * n, (long long)n, 3, bg_hwc, f64 != 0, s), "planar_to_hwc");
    });
}

int fgm_metrics_f32(const float* est, const float* gt, const float* alpha, int w, int h, int nch, double sigma,
                    int kernel_radius, double* out, void* stream) {
    return guarded([&] {
        check_dims(w, h);
        if (nch < 1) throw InvalidArgument("metrics: channels must be >= 1, got " + std::to_string(nch));
        if (!est || !gt || !alpha || !out) throw InvalidArgument("metrics: null buffer");
        // GradParams::validate (metrics.cpp:13-16), same messages
        if (!(sigma > 0.0)) throw InvalidArgument("GradParams: sigma must be > 0");
        const int r = kernel_radius > 0 ? kernel_radius : int(std::ceil(4.0 * sigma));
        if (r < 1) throw InvalidArgument("GradParams: kernel radius must be >= 1");
        require_device();
        // gaussian_derivative_kernel (metrics.cpp:61-73), host fp64
        std::vector<double> kern(size_t(2 * r + 1));
        double ramp = 0.0;
        for (int k = -r; k <= r; ++k) {
            const double g = std::exp(-(double(k) * k) / (2.0 * sigma * sigma));
            kern[size_t(k + r)] = double(k) * g;
            ramp += double(k) * k * g;
        }
        for (double& x : kern) x /= ramp;
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        const int blocks = metrics_blocks((long long)w * h);
        Arena A;
        A.reserve(al(kern.size() * sizeof(double)) + al(size_t(blocks) * 4 * sizeof(double)), s);
        double* dk = A.take<double>(kern.size());
        double* dp = A.take<double>(size_t(blocks) * 4);
        ck(cudaMemcpyAsync(dk, kern.data(), kern.size() * sizeof(double), cudaMemcpyHostToDevice, s), "H2D");
        ck(launch_metrics(est, gt, alpha, w, h, nch, dk, r, dp, blocks, s), "metrics_kernel");
        std::vector<double> part(size_t(blocks) * 4);
        ck(cudaMemcpyAsync(part.data(), dp, part.size() * sizeof(double), cudaMemcpyDeviceToHost, s), "D2H");
        ck(cudaStreamSynchronize(s), "cudaStreamSynchronize");
        for (int q = 0; q < 4; ++q) {
            double acc = 0.0;
            for (int b = 0; b < blocks; ++b) acc += part[size_t(b) * 4 + q];
            out[q] = acc;
        }
    });
}

int fgm_compose_f32(const float* fg, const float* bg, const float* alpha, int w, int h, int nch, float* out,
                    void* stream) {
    return guarded([&] {
        check_dims(w, h);
        if (nch < 1) throw InvalidArgument("compose: channels must be >= 1, got " + std::to_string(nch));
        if (!fg || !bg || !alpha || !out) throw InvalidArgument("compose: null buffer");
        require_device();
        ck(launch_compose(fg, bg, alpha, (long long)w * h, nch, out, static_cast<cudaStream_t>(stream)),
           "compose_kernel");
    });
}

int fgm_sweep_passes_f32(const float* image, const float* alpha, const float* fg_in, const float* bg_in, int w,
                         int h, int iterations, double regularization, double gradient_weight, float* fg_out,
                         float* bg_out, void* stream) {
    return fgm_sweep_passes_kernel_f32(image, alpha, fg_in, bg_in, w, h, iterations, regularization, gradient_weight,
                                       fg_out, bg_out, 0, stream);
}

int fgm_sweep_passes_kernel_f32(const float* image, const float* alpha, const float* fg_in, const float* bg_in,
                                int w, int h, int iterations, double regularization, double gradient_weight,
                                float* fg_out, float* bg_out, int kernel, void* stream) {
    return guarded([&] {
        check_dims(w, h);
        if (iterations < 1) throw InvalidArgument("MlParams: iteration counts must be >= 1");
        if (kernel < 0 || kernel > 2) throw InvalidArgument("sweep kernel must be 0 (automatic), 1 or 2");
        const bool lat = kernel != 2;  // one image: latency-bound
        const int rows = lat ? kLatBandRows : kBandRows;
        fgm_params p{regularization, gradient_weight, 1, 1, 1};
        validate(&p);
        require_device();
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        const std::vector<int> ps = passes_for(iterations);
        const long long px = (long long)w * h;
        size_t sf = 0;
        int mb = 0;
        for (int K : ps) {
            sf = std::max(sf, sweep_stream_floats(w, h, K, rows));
            mb = std::max(mb, sweep_bands(h, K, rows));
        }
        Arena A;
        A.reserve(al(sf * 4) + al(size_t(3 * mb + 1) * 4) + 2 * al(6 * size_t(px) * 4) + 256 * (ps.size() + 2) +
                      al(size_t(3 * mb) * sizeof(int2)) * ps.size(), s);
        float* stream_buf = A.take<float>(sf);
        unsigned* ctr = A.take<unsigned>(size_t(3 * mb) + 1);
        float* tmp[2] = {A.take<float>(6 * size_t(px)), A.take<float>(6 * size_t(px))};
        const float* fi = fg_in;
        const float* bi = bg_in;
        for (size_t pi = 0; pi < ps.size(); ++pi) {
            const bool last = pi + 1 == ps.size();
            SweepJob J1{};
            J1.img = image;
            J1.alpha = alpha;
            J1.fg_in = fi;
            J1.bg_in = bi;
            J1.fg_out = last ? fg_out : tmp[pi & 1];
            J1.bg_out = last ? bg_out : tmp[pi & 1] + 3 * px;
            J1.stream = stream_buf;
            J1.ipitch = J1.fpitch = J1.opitch = w;  // the caller's dense planes
            J1.istride = J1.fstride = J1.ostride = px;
            J1.w = w;
            J1.h = h;
            J1.nb = sweep_bands(h, ps[pi], rows);
            J1.band_base = 0;
            J1.vec4 = vec4_ok(J1);
            ck(cudaMemsetAsync(ctr, 0, 2 * sizeof(unsigned), s), "memset");
            SweepJob* d = A.take<SweepJob>(1);
            ck(cudaMemcpyAsync(d, &J1, sizeof(J1), cudaMemcpyHostToDevice, s), "cudaMemcpyAsync(jobs)");
            const std::vector<int2> ord = band_order({J1}, rows);
            int2* dord = A.take<int2>(ord.size());
            ck(cudaMemcpyAsync(dord, ord.data(), ord.size() * sizeof(int2), cudaMemcpyHostToDevice, s),
               "cudaMemcpyAsync(order)");
            ck(launch_stream_fill(d, 1, ps[pi], sf, s), "stream_fill_kernel");
            {
                ProfScope pr(s, 0, 64.0 * double(px));
                ck(launch_sweep_passes(ps[pi], d, dord, J1.nb, ctr, float(regularization), float(gradient_weight), lat,
                                       s),
                   "sweep_kernel");
            }
            fi = J1.fg_out;
            bi = J1.bg_out;
        }
    });
}

void fgm_debug_fault(int code) { fgm::g_sweep_fault.store(code); }


void fgm_set_spin_timeout_ms(int ms) { fgm::g_spin_timeout_ns.store((long long)std::max(ms, 1) * 1000000ll); }

int fgm_device_faults(int reset) {
    int v = -1;
    const int rc = guarded([&] {
        require_device();
        ck(cudaDeviceSynchronize(), "cudaDeviceSynchronize");
        v = read_faults();
        if (reset) ck(cudaMemset(device_fault_counter(), 0, sizeof(int)), "cudaMemset(fault counter)");
    });
    return rc ? -rc : v;
}
void fgm_set_pyramid_mode(int fused) { g_pyramid_mode.store(fused ? 1 : 0); }
void fgm_set_debug_guards(int on) { fgm::g_debug_guards.store(on ? 1 : 0); }

void fgm_profile_enable(int on) {
    std::lock_guard<std::mutex> g(g_prof_mu);
    g_prof_on = on != 0;
}

void fgm_profile_reset(void) {
    prof_drain();
    std::lock_guard<std::mutex> g(g_prof_mu);
    for (int i = 0; i < 4; ++i) {
        g_launches[i] = 0;
        g_ms[i] = 0;
        g_bytes[i] = 0;
    }
}

int fgm_kernel_stats(int which, long long* launches, double* ms, double* alg_bytes) {
    if (which < 0 || which > 3) return FGM_INVALID_ARGUMENT;
    prof_drain();
    std::lock_guard<std::mutex> g(g_prof_mu);
    if (launches) *launches = g_launches[which];
    if (ms) *ms = g_ms[which];
    if (alg_bytes) *alg_bytes = g_bytes[which];
    return FGM_OK;
}

int fgm_profile_timeline(int max, int* which, double* t0, double* t1) {
    prof_drain();
    std::lock_guard<std::mutex> g(g_prof_mu);
    const int n = int(g_timeline.size());
    for (int i = 0; i < std::min(n, max); ++i) {
        if (which) which[i] = g_timeline[size_t(i)].which;
        if (t0) t0[i] = g_timeline[size_t(i)].t0;
        if (t1) t1[i] = g_timeline[size_t(i)].t1;
    }
    return n;
}

int fgm_release_memory(void) {
    return guarded([&] {
        require_device();
        ck(cudaDeviceSynchronize(), "cudaDeviceSynchronize");
        ck(cudaMemPoolTrimTo(device_pool(), 0), "cudaMemPoolTrimTo");
    });
}

const char* fgm_last_error(void) { return fgm::g_err.c_str(); }

int fgm_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) return 0;
    return n;
}

const char* fgm_version(void) { return "fgmatte_b200 0.1.0 (sm_100a)"; }

}  // extern "C"
