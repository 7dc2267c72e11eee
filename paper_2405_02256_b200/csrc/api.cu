// eucalc C ABI — host runtime (handles, validation, capacity protocol, launches).
// See include/eucalc.h for the contract of every entry point.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <new>
#include <numeric>
#include <string>
#include <tuple>
#include <vector>

#include "eucalc_internal.cuh"

namespace eucalc {
int k3_chunk();

namespace {
thread_local std::string g_err;
thread_local int64_t g_bad = -1;
thread_local int64_t g_launches = 0;
std::atomic<int64_t> g_k2_restarts{0};  // eucalc_k2_restarts (test hook EUCALC_K2_CHK_BITS)

// ---- stage timing (eucalc_profile_*) ----
struct ProfRec {
    std::string stage;
    cudaEvent_t a, b;
    int64_t launches;
};
thread_local bool g_prof = false;
thread_local std::vector<ProfRec> g_prof_recs;
thread_local std::vector<cudaEvent_t> g_ev_pool;

cudaEvent_t ev_get() {
    if (!g_ev_pool.empty()) {
        cudaEvent_t e = g_ev_pool.back();
        g_ev_pool.pop_back();
        return e;
    }
    cudaEvent_t e = nullptr;
    cudaEventCreate(&e);
    return e;
}
struct ProfScope {
    bool on;
    cudaStream_t st;
    cudaEvent_t a = nullptr;
    int64_t l0;
    std::string stage;
    ProfScope(const char *name, cudaStream_t s) : on(g_prof), st(s), l0(g_launches), stage(name) {
        if (on) {
            a = ev_get();
            cudaEventRecord(a, st);
        }
    }
    ~ProfScope() {
        if (on) {
            cudaEvent_t b = ev_get();
            cudaEventRecord(b, st);
            g_prof_recs.push_back(ProfRec{stage, a, b, g_launches - l0});
        }
    }
};

// ---- host trace (EUCALC_HOST_TRACE=1: microseconds between marks, to stderr) ----
struct HostTrace {
    bool on = getenv("EUCALC_HOST_TRACE") != nullptr;
    std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now(), last = t0;
    const char *fn;
    std::string line;
    explicit HostTrace(const char *f) : fn(f) {}
    void mark(const char *what) {
        if (!on) return;
        const auto t = std::chrono::steady_clock::now();
        line += std::string(" ") + what + "=" +
                std::to_string(std::chrono::duration_cast<std::chrono::microseconds>(t - last).count());
        last = t;
    }
    ~HostTrace() {
        if (on) fprintf(stderr, "[trace] %s:%s us\n", fn, line.c_str());
    }
};

eucalc_status fail(eucalc_status s, const std::string &msg) {
    g_err = msg;
    return s;
}
eucalc_status cuda_fail(cudaError_t e, const char *where) {
    g_err = std::string(where) + ": " + cudaGetErrorString(e);
    return EUCALC_E_CUDA;
}
#define CK(expr)                                                 \
    do {                                                         \
        cudaError_t _e = (expr);                                 \
        if (_e != cudaSuccess) return cuda_fail(_e, #expr);      \
    } while (0)

bool is_device_ptr(const void *p) {
    if (!p) return false;
    cudaPointerAttributes at;
    cudaError_t e = cudaPointerGetAttributes(&at, p);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
}

// Page-locked host memory (cudaHostAlloc / cudaHostRegister): async copies from
// it are still in flight when cudaMemcpyAsync returns.
bool is_pinned_host_ptr(const void *p) {
    if (!p) return false;
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return at.type == cudaMemoryTypeHost;
}

// Blocks until everything enqueued on `st` so far has completed (one event
// record + wait; the rest of the stream keeps its asynchrony).
cudaError_t wait_stream_point(cudaStream_t st) {
    static thread_local cudaEvent_t ev = nullptr;
    if (!ev) {
        cudaError_t e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
        if (e != cudaSuccess) return e;
    }
    cudaError_t e = cudaEventRecord(ev, st);
    return e == cudaSuccess ? cudaEventSynchronize(ev) : e;
}

int num_sms() {
    static thread_local int n = 0;
    if (!n) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        if (n <= 0) n = 148;
    }
    return n;
}

// Keep freed stream-ordered allocations in the device's default pool (the
// default release threshold of 0 returns them to the driver at every
// synchronisation, so each later cudaMallocAsync became a full allocation:
// ~1 ms per call measured on the bench step).
void keep_pool() {
    static std::mutex mu;
    static bool done[64] = {};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return;
    std::lock_guard<std::mutex> lk(mu);
    if (done[dev]) return;
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        uint64_t thr = UINT64_MAX;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    cudaGetLastError();
    done[dev] = true;
}

// Per-(thread, stream) device scratch arena for the small per-call buffers
// (look-back flags, tickets, counts, slabs, kbar tables): one allocation that
// only grows, carved per call. Reuse is stream-ordered: a later call on the same
// stream runs after the kernels of the earlier one. Never released (bounded by
// the largest call).
struct Arena {
    void *p = nullptr;
    size_t cap = 0;
};
thread_local std::map<cudaStream_t, Arena> g_arenas;

// Carves `sizes` (256-byte aligned) out of the arena of `st`; false on allocation failure.
bool arena_take(cudaStream_t st, const std::vector<size_t> &sizes, std::vector<void *> &out) {
    size_t total = 0;
    for (size_t b : sizes) total += (b + 255) / 256 * 256;
    Arena &ar = g_arenas[st];
    if (total > ar.cap) {
        if (ar.p) cudaFreeAsync(ar.p, st);
        ar.p = nullptr;
        ar.cap = 0;
        const size_t want = std::max<size_t>(total, size_t(1) << 20);
        if (cudaMallocAsync(&ar.p, want, st) != cudaSuccess) {
            cudaGetLastError();
            return false;
        }
        ar.cap = want;
    }
    out.clear();
    size_t off = 0;
    for (size_t b : sizes) {
        out.push_back(b ? (unsigned char *)ar.p + off : nullptr);
        off += (b + 255) / 256 * 256;
    }
    return true;
}

// Releases (stream-ordered) an arena that one large call pushed past
// kArenaKeep, so that memory is not held for the life of the stream.
constexpr size_t kArenaKeep = size_t(256) << 20;
void arena_trim(cudaStream_t st) {
    auto it = g_arenas.find(st);
    if (it == g_arenas.end() || it->second.cap <= kArenaKeep) return;
    cudaFreeAsync(it->second.p, st);
    g_arenas.erase(it);
}

int bits_for(int64_t v) {  // bits to hold 0..v
    int b = 1;
    while ((int64_t(1) << b) <= v) ++b;
    return b;
}

template <typename T>
__global__ void maxabs_kernel(const T *p, int64_t n, unsigned long long *out) {
    unsigned long long m = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        long long v = (long long)p[i];
        unsigned long long a = (unsigned long long)(v < 0 ? -v : v);
        m = a > m ? a : m;
    }
    for (int d = 16; d; d >>= 1) {
        unsigned long long o = __shfl_xor_sync(0xffffffffu, m, d);
        m = o > m ? o : m;
    }
    if ((threadIdx.x & 31) == 0) atomicMax(out, m);
}

struct DirPlan {
    std::vector<int32_t> host;  // [D][n]
    std::vector<DirInfo> info;
    std::vector<int32_t> csum;
    std::vector<int> orthant;
    int R_max = 0;
    int dp = 0;  // all directions fit int8 and the complex is byte-aligned
    int64_t U0 = 0, U1 = 0;  // range of u = 2H - L*csum over all directions (K3 kbar table)
    // per antipodal pair q: the height ranges R of its directions, sorted, with prefix sums
    std::vector<std::vector<int64_t>> Rq, preq;
    uint64_t id = 0;         // unique per plan (bound cache key)
};

// Max number of vertices on one lattice height level {p : sum xs_k p_k = h}:
// along two axes j, k the solutions step by (xs_k, -xs_j) / gcd, so a line holds
// at most min((M_j-1) / |xs_k/g|, (M_k-1) / |xs_j/g|) + 1 points; in 3-D a level
// set is at most (extent of the third axis) lines. Bounds every histogram bin's
// record count (K2's packed-bin test per direction).
int64_t level_points(const Complex *cx, const DirInfo &di) {
    const int n = cx->ndim;
    auto line2 = [&](int j, int k) -> int64_t {
        const int64_t a = std::llabs((int64_t)di.xs[j]), b = std::llabs((int64_t)di.xs[k]);
        if (a == 0 || b == 0) return int64_t(1);  // an extent-1 axis (scale 0): one point per height
        const int64_t g = std::gcd(a, b);
        return std::min((cx->M[j] - 1) / (b / g), (cx->M[k] - 1) / (a / g)) + 1;
    };
    if (n == 2) return line2(0, 1);
    return std::min({cx->M[0] * line2(1, 2), cx->M[1] * line2(0, 2), cx->M[2] * line2(0, 1)});
}

eucalc_status plan_dirs(const Complex *cx, const int32_t *dirs, int64_t D, cudaStream_t st, DirPlan &p) {
    if (D < 0) return fail(EUCALC_E_ARG, "D < 0");
    if (D > 0 && !dirs) return fail(EUCALC_E_ARG, "dirs is NULL");
    const int n = cx->ndim;
    p.host.resize((size_t)D * n);
    if (D > 0) {
        if (is_device_ptr(dirs)) {
            CK(cudaMemcpyAsync(p.host.data(), dirs, sizeof(int32_t) * D * n, cudaMemcpyDeviceToHost, st));
            CK(cudaStreamSynchronize(st));
        } else {
            memcpy(p.host.data(), dirs, sizeof(int32_t) * D * n);
        }
    }
    p.info.resize(D);
    p.csum.resize(D);
    p.orthant.resize(D);
    p.R_max = 1;
    const int full = (1 << n) - 1;
    for (int64_t d = 0; d < D; ++d) {
        DirInfo di{};
        int e = 0;
        int64_t lo = 0, hi = 0, cs = 0;
        for (int k = 0; k < n; ++k) {
            const int64_t xi = p.host[d * n + k];
            if (xi == 0) {
                g_bad = d;
                return fail(EUCALC_E_NONGENERIC, "direction " + std::to_string(d) + " has a zero coordinate (P:105)");
            }
            if (xi > 0) e |= 1 << k;
            const int64_t xs = xi * cx->scale[k];
            if (xs > INT32_MAX || xs < INT32_MIN) return fail(EUCALC_E_RANGE, "scaled direction overflows int32");
            di.xs[k] = (int)xs;
            const int64_t ext = xs * (cx->M[k] - 1);
            if (ext < 0) lo += ext; else hi += ext;
            if (cx->M[k] > 1) cs += xi;
        }
        if (lo < -(int64_t(1) << 30) || hi > (int64_t(1) << 30))
            return fail(EUCALC_E_RANGE, "lattice heights exceed the int32 kernel range");
        di.hlo = (int)lo;
        di.R = (int)(hi - lo + 1);
        const bool rep = ((e >> (n - 1)) & 1) == 0;
        di.q = rep ? e : (e ^ full);
        di.swap = rep ? 0 : 1;
        p.info[d] = di;
        p.csum[d] = (int32_t)cs;
        p.info[d].lcsum = cx->L * cs;
        p.orthant[d] = e;
        p.R_max = std::max(p.R_max, di.R);
        const int64_t Lc = cx->L * cs, ulo = 2 * lo - Lc, uhi = 2 * hi - Lc;
        p.U0 = d == 0 ? ulo : std::min(p.U0, ulo);
        p.U1 = d == 0 ? uhi : std::max(p.U1, uhi);
        bool fits8 = true;
        uint32_t x8 = 0;
        for (int k = 0; k < n; ++k) {
            fits8 = fits8 && di.xs[k] >= -127 && di.xs[k] <= 127;
            x8 |= (uint32_t)(di.xs[k] & 0xff) << (8 * (n - 1 - k));
        }
        p.info[d].xs8 = (int)x8;
        p.info[d].line = (int)std::min<int64_t>(level_points(cx, p.info[d]), INT32_MAX);
        if (d == 0) p.dp = cx->aligned;
        if (!fits8) p.dp = 0;
    }
    const int Q = 1 << (n - 1);
    p.Rq.assign(Q, {});
    p.preq.assign(Q, {});
    for (int64_t d = 0; d < D; ++d) p.Rq[p.info[d].q].push_back(p.info[d].R);
    for (int q = 0; q < Q; ++q) {
        std::sort(p.Rq[q].begin(), p.Rq[q].end());
        p.preq[q].assign(p.Rq[q].size() + 1, 0);
        for (size_t i = 0; i < p.Rq[q].size(); ++i) p.preq[q][i + 1] = p.preq[q][i] + p.Rq[q][i];
    }
    static std::atomic<uint64_t> next_id{1};
    p.id = next_id++;
    return EUCALC_OK;
}

// ---- direction plans, cached with their device copies ------------------------
// A plan holds the host DirInfo and the device arrays K2/K3 read (DirInfo,
// csum, orthant-grouped order and tiles). Re-using a direction set (the common
// case: many batches, one set of directions) then costs no host->device copy
// — a pageable cudaMemcpyAsync would synchronise the stream.
struct PlanEntry {
    std::vector<int32_t> key;
    int ndim = 0, aligned = 0, dev = 0;
    int64_t M[kMaxN] = {0, 0, 0}, scale[kMaxN] = {0, 0, 0};
    DirPlan p;
    std::vector<int32_t> order, tstart, tlen;
    DirInfo *d_info = nullptr;
    int32_t *d_csum = nullptr, *d_order = nullptr, *d_ts = nullptr, *d_tl = nullptr;
    uint64_t stamp = 0;
    // K2 unit path (k2_unit): directions grouped by (pair, side) into units, and
    // each direction's staging slot within an image; built on first use
    std::mutex unit_mu;
    bool units_built = false;
    int64_t nunits = 0, stage_img = 0;
    int4 *d_units = nullptr;
    int32_t *d_unit_dirs = nullptr;
    int64_t *d_stage_base = nullptr;
    int32_t *d_dir_by_R = nullptr;  // directions by decreasing R (slot mode's segment order)
    // the same directions in units balanced for a single image (plan_units_balanced)
    bool bal_built = false;
    int64_t bal_nunits = 0;
    int4 *d_bal_units = nullptr;
    int32_t *d_bal_unit_dirs = nullptr;
    ~PlanEntry() {
        cudaFree(d_units);
        cudaFree(d_unit_dirs);
        cudaFree(d_bal_units);
        cudaFree(d_bal_unit_dirs);
        cudaFree(d_stage_base);
        cudaFree(d_dir_by_R);
        // cudaFree synchronises the device, so no in-flight kernel still reads these
        cudaFree(d_info);
        cudaFree(d_csum);
        cudaFree(d_order);
        cudaFree(d_ts);
        cudaFree(d_tl);
    }
};
std::mutex g_plan_mu;
std::vector<std::shared_ptr<PlanEntry>> g_plans;
uint64_t g_plan_clock = 0;
constexpr size_t kMaxPlans = 16;

eucalc_status get_plan(const Complex *cx, const int32_t *dirs, int64_t D, cudaStream_t st,
                       std::shared_ptr<PlanEntry> &out) {
    if (D < 0) return fail(EUCALC_E_ARG, "D < 0");
    if (D > 0 && !dirs) return fail(EUCALC_E_ARG, "dirs is NULL");
    const int n = cx->ndim;
    std::vector<int32_t> h((size_t)D * n);
    if (D > 0) {
        if (is_device_ptr(dirs)) {
            CK(cudaMemcpyAsync(h.data(), dirs, sizeof(int32_t) * D * n, cudaMemcpyDeviceToHost, st));
            CK(cudaStreamSynchronize(st));
        } else {
            memcpy(h.data(), dirs, sizeof(int32_t) * D * n);
        }
    }
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lk(g_plan_mu);
    for (auto &e : g_plans) {
        if (e->ndim == n && e->dev == dev && e->aligned == cx->aligned && e->key == h &&
            std::equal(e->M, e->M + n, cx->M) && std::equal(e->scale, e->scale + n, cx->scale)) {
            e->stamp = ++g_plan_clock;
            out = e;
            return EUCALC_OK;
        }
    }
    auto e = std::make_shared<PlanEntry>();
    eucalc_status s = plan_dirs(cx, h.data(), D, st, e->p);
    if (s != EUCALC_OK) return s;
    e->key = std::move(h);
    e->ndim = n;
    e->dev = dev;
    e->aligned = cx->aligned;
    std::copy(cx->M, cx->M + n, e->M);
    std::copy(cx->scale, cx->scale + n, e->scale);
    // HT tiles: directions grouped by orthant (Lemma 3), <= 512 per tile
    e->order.resize(D);
    std::iota(e->order.begin(), e->order.end(), 0);
    // tile key: orthant (same critical list, Lemma 3) and the parity of L*csum
    // (the parity of u = 2H - L*csum, which selects one half of K3's kbar table)
    auto key = [&](int32_t d) { return e->p.orthant[d] * 2 + (int)((cx->L * (int64_t)e->p.csum[d]) & 1); };
    std::stable_sort(e->order.begin(), e->order.end(), [&](int32_t x, int32_t y) { return key(x) < key(y); });
    for (int64_t i = 0; i < D;) {
        int64_t j = i;
        while (j < D && key(e->order[j]) == key(e->order[i]) && j - i < 512) ++j;
        e->tstart.push_back((int32_t)i);
        e->tlen.push_back((int32_t)(j - i));
        i = j;
    }
    if (D > 0) {
        const size_t nt = e->tstart.size();
        CK(cudaMalloc(&e->d_info, sizeof(DirInfo) * D));
        CK(cudaMalloc(&e->d_csum, sizeof(int32_t) * D));
        CK(cudaMalloc(&e->d_order, sizeof(int32_t) * D));
        CK(cudaMalloc(&e->d_ts, sizeof(int32_t) * nt));
        CK(cudaMalloc(&e->d_tl, sizeof(int32_t) * nt));
        CK(cudaMemcpy(e->d_info, e->p.info.data(), sizeof(DirInfo) * D, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(e->d_csum, e->p.csum.data(), sizeof(int32_t) * D, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(e->d_order, e->order.data(), sizeof(int32_t) * D, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(e->d_ts, e->tstart.data(), sizeof(int32_t) * nt, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(e->d_tl, e->tlen.data(), sizeof(int32_t) * nt, cudaMemcpyHostToDevice));
    }
    e->stamp = ++g_plan_clock;
    if (g_plans.size() >= kMaxPlans) {
        auto it = std::min_element(g_plans.begin(), g_plans.end(),
                                   [](const auto &x, const auto &y) { return x->stamp < y->stamp; });
        g_plans.erase(it);
    }
    g_plans.push_back(e);
    out = e;
    return EUCALC_OK;
}

// Units of the K2 unit path for a direction plan: the directions of each (pair,
// side) group, largest R first, packed greedily into units of at most
// k2_unit_max() directions whose 128-padded R sum fits k2_unit_words(); units
// with more directions first. Staging slot of direction d: sum of R over d' < d.
eucalc_status plan_units(PlanEntry &pe) {
    std::lock_guard<std::mutex> lk(pe.unit_mu);
    if (pe.units_built) return EUCALC_OK;
    const DirPlan &p = pe.p;
    const int64_t D = (int64_t)p.info.size();
    std::vector<int32_t> idx(D);
    std::iota(idx.begin(), idx.end(), 0);
    auto key = [&](int32_t d) { return p.info[d].q * 2 + p.info[d].swap; };
    std::stable_sort(idx.begin(), idx.end(), [&](int32_t x, int32_t y) {
        if (key(x) != key(y)) return key(x) < key(y);
        return p.info[x].R > p.info[y].R;
    });
    std::vector<int4> units;
    std::vector<int32_t> dirs_out;
    int gmax = k2_unit_max();
    const int words = k2_unit_words();
    if (const char *v = getenv("EUCALC_K2_UNIT_G")) gmax = std::max(1, std::min(gmax, atoi(v)));  // measurement hook
    for (int64_t i = 0; i < D;) {
        int4 u{(int)dirs_out.size(), 0, p.info[idx[i]].q, p.info[idx[i]].swap};
        int64_t off = 0;
        while (i < D && u.y < gmax && key(idx[i]) == u.z * 2 + u.w) {
            const int64_t rp = (p.info[idx[i]].R + 127) / 128 * 128;
            if (u.y > 0 && off + rp > words) break;
            off += rp;
            dirs_out.push_back(idx[i]);
            ++u.y;
            ++i;
        }
        units.push_back(u);
    }
    std::stable_sort(units.begin(), units.end(), [](const int4 &x, const int4 &y) { return x.y > y.y; });
    std::vector<int64_t> base(D);
    int64_t acc = 0;
    for (int64_t d = 0; d < D; ++d) {
        base[d] = acc;
        acc += p.info[d].R;
    }
    if (!units.empty()) {
        CK(cudaMalloc(&pe.d_units, sizeof(int4) * units.size()));
        CK(cudaMalloc(&pe.d_unit_dirs, sizeof(int32_t) * dirs_out.size()));
        CK(cudaMalloc(&pe.d_stage_base, sizeof(int64_t) * D));
        CK(cudaMemcpy(pe.d_units, units.data(), sizeof(int4) * units.size(), cudaMemcpyHostToDevice));
        CK(cudaMemcpy(pe.d_unit_dirs, dirs_out.data(), sizeof(int32_t) * dirs_out.size(), cudaMemcpyHostToDevice));
        CK(cudaMemcpy(pe.d_stage_base, base.data(), sizeof(int64_t) * D, cudaMemcpyHostToDevice));
        std::vector<int32_t> by_r(D);
        std::iota(by_r.begin(), by_r.end(), 0);
        std::stable_sort(by_r.begin(), by_r.end(), [&](int32_t x, int32_t y) { return p.info[x].R > p.info[y].R; });
        CK(cudaMalloc(&pe.d_dir_by_R, sizeof(int32_t) * D));
        CK(cudaMemcpy(pe.d_dir_by_R, by_r.data(), sizeof(int32_t) * D, cudaMemcpyHostToDevice));
    }
    pe.nunits = (int64_t)units.size();
    pe.stage_img = acc;
    pe.units_built = true;
    return EUCALC_OK;
}

// Units for ONE image on `sms` SMs. Every unit streams its whole list, so units of
// kUnitMax directions minimise the work, but U units of equal cost on P SMs take
// ceil(U / P) waves (config 4: 256 units on 148 SMs = 2 waves, the second 73% full).
// Here the unit count is raised to the next multiple of P by giving the (pair, side)
// groups with the most directions per unit one more unit each, and a group's
// directions are spread evenly over its units (sizes differ by at most one): 296
// units of 4 or 3 directions take one wave of each (cost of a unit ~ 0.11 + 0.22 G of
// a 4-direction unit: 1.78 against 2.0). Only taken when it lowers that estimate;
// with several images the light images' units fill the last wave instead (plan_units).
// Built after plan_units (shares its staging slots). bal_nunits == 0: no gain.
eucalc_status plan_units_balanced(PlanEntry &pe, int sms) {
    std::lock_guard<std::mutex> lk(pe.unit_mu);
    if (pe.bal_built) return EUCALC_OK;
    pe.bal_built = true;
    const DirPlan &p = pe.p;
    const int64_t D = (int64_t)p.info.size();
    const int gmax = k2_unit_max(), words = k2_unit_words();
    if (pe.nunits <= sms || pe.nunits % sms == 0) return EUCALC_OK;
    std::vector<int32_t> idx(D);
    std::iota(idx.begin(), idx.end(), 0);
    auto key = [&](int32_t d) { return p.info[d].q * 2 + p.info[d].swap; };
    std::stable_sort(idx.begin(), idx.end(), [&](int32_t x, int32_t y) {
        if (key(x) != key(y)) return key(x) < key(y);
        return p.info[x].R > p.info[y].R;
    });
    struct Group { int64_t i0, n, u; };
    std::vector<Group> groups;
    for (int64_t i = 0; i < D;) {
        int64_t j = i;
        while (j < D && key(idx[j]) == key(idx[i])) ++j;
        groups.push_back({i, j - i, (j - i + gmax - 1) / gmax});
        i = j;
    }
    int64_t U = 0;
    for (const Group &g : groups) U += g.u;
    const int64_t target = (U + sms - 1) / sms * sms;
    while (U < target) {  // one more unit for the group with the most directions per unit
        Group *best = nullptr;
        for (Group &g : groups)
            if (g.u < g.n && (!best || g.n * best->u > best->n * g.u)) best = &g;
        if (!best) break;
        ++best->u;
        ++U;
    }
    std::vector<int4> units;
    std::vector<int32_t> dirs_out;
    for (const Group &g : groups) {
        int64_t i = g.i0;
        for (int64_t k = 0; k < g.u; ++k) {
            // the larger units take the directions with the smaller R (sorted by decreasing R)
            const int64_t sz = g.n / g.u + (k >= g.u - g.n % g.u ? 1 : 0);
            int4 u{(int)dirs_out.size(), 0, p.info[idx[g.i0]].q, p.info[idx[g.i0]].swap};
            int64_t off = 0;
            for (int64_t t = 0; t < sz; ++t, ++i) {
                off += (p.info[idx[i]].R + 127) / 128 * 128;
                dirs_out.push_back(idx[i]);
                ++u.y;
            }
            if (off > words || u.y > gmax) return EUCALC_OK;  // does not fit shared memory: keep plan_units' units
            units.push_back(u);
        }
    }
    // estimated makespans (units of a kUnitMax-direction unit), heaviest units first
    auto cost = [&](int G) { return 0.107 + 0.223 * G * 4.0 / gmax; };
    std::stable_sort(units.begin(), units.end(), [](const int4 &x, const int4 &y) { return x.y > y.y; });
    std::vector<double> load(sms, 0.0);
    for (const int4 &u : units) *std::min_element(load.begin(), load.end()) += cost(u.y);
    const double bal = *std::max_element(load.begin(), load.end());
    const double plain = (double)((pe.nunits + sms - 1) / sms) * cost(gmax);
    if (bal >= 0.97 * plain) return EUCALC_OK;
    CK(cudaMalloc(&pe.d_bal_units, sizeof(int4) * units.size()));
    CK(cudaMalloc(&pe.d_bal_unit_dirs, sizeof(int32_t) * dirs_out.size()));
    CK(cudaMemcpy(pe.d_bal_units, units.data(), sizeof(int4) * units.size(), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(pe.d_bal_unit_dirs, dirs_out.data(), sizeof(int32_t) * dirs_out.size(), cudaMemcpyHostToDevice));
    pe.bal_nunits = (int64_t)units.size();
    return EUCALC_OK;
}

// Writes `gen` to a host-mapped word after everything before it on the stream
// (the read-back copies): the host polls that word with plain loads instead of
// cudaEventSynchronize, whose wake-up took ~60 us on the GPU boxes' VM.
__global__ void k1_signal(volatile unsigned *flag, unsigned gen) {
    __threadfence_system();
    *flag = gen;
}

eucalc_status sync_counts(Critical *cr, cudaStream_t st) {
    std::lock_guard<std::mutex> lk(cr->mu);
    if (cr->have_host) return EUCALC_OK;
    (void)st;
    const Complex *cx = cr->cx;
    const int64_t nc = cx->batch * cr->Q;
    const int64_t ns = cx->batch * (1 << cx->ndim) * 2 + 2 * nc;
    cr->h_count = new (std::nothrow) int64_t[nc];
    cr->h_stats = new (std::nothrow) int64_t[ns];
    if (!cr->h_count || !cr->h_stats) return fail(EUCALC_E_NOMEM, "host alloc");
    // the read-back was enqueued right after K1 into pinned memory: wait for it only
    // (poll the signal word; the event still decides on errors and when no word was set up)
    bool landed = false;
    if (cr->pinned_flag_off) {
        const volatile unsigned *f = (const volatile unsigned *)((unsigned char *)cr->pinned + cr->pinned_flag_off);
        for (uint64_t n = 1;; ++n) {
            if (*f == 1u) {
                landed = true;
                break;
            }
            if ((n & 4095) == 0) {
                const cudaError_t q = cudaEventQuery(cr->k1_done);
                if (q != cudaErrorNotReady) break;
            }
        }
    }
    if (!landed) CK(cudaEventSynchronize(cr->k1_done));
    const int32_t *c = (const int32_t *)cr->pinned;
    memcpy(cr->h_stats, (const unsigned char *)cr->pinned + cr->pinned_stats_off, sizeof(int64_t) * ns);
    cr->max_count = 0;
    for (int64_t i = 0; i < nc; ++i) {
        cr->h_count[i] = c[i];
        cr->max_count = std::max<int64_t>(cr->max_count, c[i]);
    }
    cr->max_abs_sum = 0;
    cr->max_rec = 0;
    const int64_t *abs_sum = cr->h_stats + cx->batch * (1 << cx->ndim) * 2;
    for (int64_t i = 0; i < nc; ++i) {
        cr->max_abs_sum = std::max<int64_t>(cr->max_abs_sum, abs_sum[i]);
        cr->max_rec = std::max<int64_t>(cr->max_rec, abs_sum[nc + i]);
    }
    cr->have_host = true;
    return EUCALC_OK;
}

// sum over (image, direction) of min(list length, R_d), in O(batch * Q * log D):
// per pair, the directions' R sorted with prefix sums.
eucalc_status bounds(Critical *cr, const DirPlan &p, cudaStream_t st, int64_t &bound) {
    eucalc_status s = sync_counts(cr, st);
    if (s != EUCALC_OK) return s;
    std::lock_guard<std::mutex> lk(cr->mu);
    if (cr->bound_plan == p.id && p.id) {  // same critical handle and direction plan
        bound = cr->bound_val;
        return EUCALC_OK;
    }
    bound = 0;
    for (int q = 0; q < cr->Q && q < (int)p.Rq.size(); ++q) {
        const std::vector<int64_t> &R = p.Rq[q], &pre = p.preq[q];
        if (R.empty()) continue;
        for (int64_t b = 0; b < cr->cx->batch; ++b) {
            const int64_t c = cr->h_count[b * cr->Q + q];
            const size_t k = std::upper_bound(R.begin(), R.end(), c) - R.begin();  // R[<k] <= c
            bound += pre[k] + (int64_t)(R.size() - k) * c;
        }
    }
    cr->bound_plan = p.id;
    cr->bound_val = bound;
    return EUCALC_OK;
}

// Every record at one lattice height lies on a distinct line along any axis k
// with M_k > 1 (the height is strictly monotone along it), so a bin holds at
// most nvert / max_k M_k records; with |a|+|b| <= max_rec per record this
// bounds every bin sum of Delta^- and of J.
int64_t bin_sum_bound(const Critical *cr) {
    const Complex *cx = cr->cx;
    int64_t mmax = 1;
    for (int k = 0; k < cx->ndim; ++k) mmax = std::max<int64_t>(mmax, cx->M[k]);
    const int64_t per_bin = std::max<int64_t>(1, cx->nvert / mmax);
    return std::min<int64_t>(cr->max_abs_sum, per_bin * cr->max_rec);
}

}  // namespace

void count_launch(int n) { g_launches += n; }

namespace {
struct PrepKey {
    const void *fn;
    int threads;
    size_t smem;
    int dev;
    bool operator<(const PrepKey &o) const {
        return std::tie(fn, threads, smem, dev) < std::tie(o.fn, o.threads, o.smem, o.dev);
    }
};
std::mutex g_prep_mu;
std::map<PrepKey, int> g_prep_occ;
std::map<std::pair<const void *, int>, size_t> g_prep_smem;
}  // namespace

cudaError_t prepare_kernel(const void *fn, int threads, size_t smem, int *occ) {
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lk(g_prep_mu);
    auto it = g_prep_occ.find(PrepKey{fn, threads, smem, dev});
    if (it != g_prep_occ.end()) {
        if (occ) *occ = it->second;
        return cudaSuccess;
    }
    size_t &cur = g_prep_smem[{fn, dev}];
    if (smem > cur) {
        cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        cur = smem;
    }
    int o = 0;
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, fn, threads, smem);
    if (e != cudaSuccess) return e;
    g_prep_occ[PrepKey{fn, threads, smem, dev}] = o;
    if (occ) *occ = o;
    return cudaSuccess;
}

namespace {
std::mutex g_pin_mu;
std::multimap<size_t, void *> g_pin_free;
}  // namespace

void *pinned_get(size_t bytes, size_t *cap) {
    size_t c = 256;
    while (c < bytes) c <<= 1;
    {
        std::lock_guard<std::mutex> lk(g_pin_mu);
        auto it = g_pin_free.find(c);
        if (it != g_pin_free.end()) {
            void *p = it->second;
            g_pin_free.erase(it);
            *cap = c;
            return p;
        }
    }
    void *p = nullptr;
    if (cudaHostAlloc(&p, c, cudaHostAllocDefault) != cudaSuccess) return nullptr;
    *cap = c;
    return p;
}

void pinned_put(void *p, size_t cap) {
    if (!p) return;
    std::lock_guard<std::mutex> lk(g_pin_mu);
    g_pin_free.emplace(cap, p);
}

// K1 launch arguments of a critical handle (the count/emit passes at creation,
// the per-orthant statistics on demand).
K1Args k1_args(const Critical *cr) {
    const Complex *cx = cr->cx;
    const int n = cx->ndim;
    K1Args a{};
    a.img = cx->d_img;
    a.dtype = cx->dtype;
    a.construction = cx->construction;
    a.ndim = n;
    a.batch = cx->batch;
    a.npix = cx->npix;
    a.vcap = cr->vcap;
    for (int k = 0; k < n; ++k) {
        a.m[k] = (int)cx->m[k];
        a.M[k] = (int)cx->M[k];
        a.sh[k] = cx->sh[k];
    }
    int TX, TY, TZ, W;
    k1_geometry(n, cx->M, cx->dtype, cx->construction, &TX, &TY, &TZ, &W);
    a.TX = cr->TX;
    a.TY = cr->TY;
    a.TZ = cr->TZ;
    a.W = W;
    a.walk = k1_walk(n, cx->M, cx->batch, cr->TX, cr->TY);
    a.tiles_x = cr->tiles_x;
    a.tiles_y = cr->tiles_y;
    a.tiles_z = cr->tiles_z;
    a.rec = cr->d_rec;
    a.wide = cr->wide;
    a.count = cr->d_count;
    a.tile_off = cr->d_tile_off;
    a.stats = cr->d_stats;
    a.abs_sum = cr->d_stats + cx->batch * (1 << n) * 2;
    a.max_rec = a.abs_sum + cx->batch * cr->Q;
    a.Q = cr->Q;
    return a;
}

}  // namespace eucalc

using namespace eucalc;

struct eucalc_complex : Complex {};
struct eucalc_critical : Critical {};

extern "C" {

const char *eucalc_status_string(eucalc_status s) {
    switch (s) {
    case EUCALC_OK: return "ok";
    case EUCALC_E_ARG: return "invalid argument";
    case EUCALC_E_NOMEM: return "out of memory";
    case EUCALC_E_CUDA: return "CUDA error";
    case EUCALC_E_NONGENERIC: return "non-generic direction (zero coordinate)";
    case EUCALC_E_CAPACITY: return "output capacity too small";
    case EUCALC_E_RANGE: return "value range exceeded";
    case EUCALC_E_STATE: return "invalid handle";
    }
    return "unknown status";
}
const char *eucalc_last_error(void) { return g_err.c_str(); }

void eucalc_profile_enable(int on) {
    for (auto &r : g_prof_recs) {
        cudaEventSynchronize(r.b);
        g_ev_pool.push_back(r.a);
        g_ev_pool.push_back(r.b);
    }
    g_prof_recs.clear();
    g_prof = on != 0;
}

int eucalc_profile_read(const char *stage, double *ms, int64_t *launches) {
    double t = 0;
    int64_t n = 0;
    for (auto &r : g_prof_recs) {
        if (stage && r.stage != stage) continue;
        cudaEventSynchronize(r.b);
        float x = 0;
        cudaEventElapsedTime(&x, r.a, r.b);
        t += x;
        n += r.launches;
    }
    if (ms) *ms = t;
    if (launches) *launches = n;
    return 0;
}
int eucalc_profile_span(const char *stage, double *ms) {
    // first start to last end over the recorded launches of `stage` (they may sit
    // on different streams and overlap): event timestamps share one GPU clock
    bool any = false;
    float lo = 0, hi = 0;
    cudaEvent_t ref = nullptr;
    for (auto &r : g_prof_recs) {
        if (stage && r.stage != stage) continue;
        cudaEventSynchronize(r.b);
        if (!ref) ref = r.a;
        float a = 0, b = 0;
        cudaEventElapsedTime(&a, ref, r.a);
        cudaEventElapsedTime(&b, ref, r.b);
        lo = any ? std::min(lo, a) : a;
        hi = any ? std::max(hi, b) : b;
        any = true;
    }
    if (ms) *ms = any ? (double)(hi - lo) : 0.0;
    return 0;
}

int64_t eucalc_last_bad_index(void) { return g_bad; }
int64_t eucalc_launch_count(int reset) {
    int64_t v = g_launches;
    if (reset) g_launches = 0;
    return v;
}
int64_t eucalc_k2_restarts(int reset) {
    int64_t v = g_k2_restarts.load();
    if (reset) g_k2_restarts = 0;
    return v;
}

eucalc_status eucalc_build_complex(const void *img, int dtype, int ndim, const int64_t *shape, int64_t batch,
                                   int construction, void *stream, eucalc_complex **out) {
    if (!out) return fail(EUCALC_E_ARG, "out is NULL");
    *out = nullptr;
    if (!img || !shape) return fail(EUCALC_E_ARG, "img/shape is NULL");
    if (dtype < EUCALC_U8 || dtype > EUCALC_I32) return fail(EUCALC_E_ARG, "bad dtype");
    if (ndim != 2 && ndim != 3) return fail(EUCALC_E_ARG, "ndim must be 2 or 3");
    if (batch < 1) return fail(EUCALC_E_ARG, "batch < 1");
    if (construction != EUCALC_VERTEX && construction != EUCALC_TOP) return fail(EUCALC_E_ARG, "bad construction");
    cudaStream_t st = (cudaStream_t)stream;
    keep_pool();
    eucalc_complex *cx = new (std::nothrow) eucalc_complex();
    if (!cx) return fail(EUCALC_E_NOMEM, "host alloc");
    cx->ndim = ndim;
    cx->dtype = dtype;
    cx->construction = construction;
    cx->batch = batch;
    cx->npix = 1;
    cx->nvert = 1;
    for (int k = 0; k < ndim; ++k) {
        if (shape[k] < 1 || shape[k] > (1 << 20)) {
            delete cx;
            return fail(EUCALC_E_ARG, "shape out of range");
        }
        cx->m[k] = shape[k];
        cx->M[k] = construction == EUCALC_VERTEX ? shape[k] : shape[k] + 1;
        cx->npix *= cx->m[k];
        cx->nvert *= cx->M[k];
    }
    if (cx->nvert > INT32_MAX) {
        delete cx;
        return fail(EUCALC_E_ARG, "image too large");
    }
    // packed coordinates: axis n-1 in the low bits. Byte-aligned fields (16-bit
    // halves in 2-D, bytes in 3-D) when the extents allow, so the height is one
    // dp2a / dp4a instruction against the direction's packed int8 coordinates.
    int sh = 0;
    bool al2 = ndim == 2 && cx->M[0] <= 65536 && cx->M[1] <= 65536;
    bool al3 = ndim == 3 && cx->M[0] <= 256 && cx->M[1] <= 256 && cx->M[2] <= 256;
    cx->aligned = al2 ? 2 : al3 ? 3 : 0;
    for (int k = ndim - 1; k >= 0; --k) {
        int bw = al2 ? 16 : al3 ? 8 : bits_for(cx->M[k] - 1);
        cx->sh[k] = sh;
        cx->msk[k] = (uint32_t)((1ull << bw) - 1);
        sh += bw;
    }
    if (sh > 32) {
        delete cx;
        return fail(EUCALC_E_ARG, "packed vertex coordinates need more than 32 bits");
    }
    // height scale (E10): L = lcm of (M_i - 1) > 0
    int64_t L = 1;
    for (int k = 0; k < ndim; ++k)
        if (cx->M[k] > 1) L = L / std::gcd(L, cx->M[k] - 1) * (cx->M[k] - 1);
    cx->L = L;
    for (int k = 0; k < ndim; ++k) cx->scale[k] = cx->M[k] > 1 ? L / (cx->M[k] - 1) : 0;
    const size_t esz = dtype == EUCALC_U8 ? 1 : dtype == EUCALC_I16 ? 2 : 4;
    const size_t bytes = esz * (size_t)(cx->npix * batch);
    cudaError_t e = cudaMallocAsync(&cx->d_img, bytes, st);
    if (e != cudaSuccess) {
        delete cx;
        return cuda_fail(e, "cudaMallocAsync(image)");
    }
    const bool dev_src = is_device_ptr(img);
    e = cudaMemcpyAsync(cx->d_img, img, bytes, dev_src ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, st);
    if (dtype == EUCALC_U8) {
        // |w| <= 255 by type: no reduction. A host source may be freed by the
        // caller when this call returns (eucalc.h): from pageable memory the copy
        // has consumed the buffer on return, from pinned memory it is still in
        // flight, so wait for it (the stream's earlier work included).
        if (e == cudaSuccess && !dev_src && is_pinned_host_ptr(img)) e = wait_stream_point(st);
        if (e != cudaSuccess) {
            cudaFreeAsync(cx->d_img, st);
            delete cx;
            return cuda_fail(e, "build_complex");
        }
        cx->max_abs_w = 255;
        cx->owner_stream = st;
        *out = cx;
        return EUCALC_OK;
    }
    unsigned long long *d_max = nullptr;
    if (e == cudaSuccess) e = cudaMallocAsync(&d_max, sizeof(unsigned long long), st);
    if (e == cudaSuccess) e = cudaMemsetAsync(d_max, 0, sizeof(unsigned long long), st);
    if (e == cudaSuccess) {
        const int64_t n = cx->npix * batch;
        ProfScope ps("build", st);
        const unsigned g = (unsigned)std::min<int64_t>(4 * 148, (n + 255) / 256);
        if (dtype == EUCALC_U8) maxabs_kernel<<<g, 256, 0, st>>>((const uint8_t *)cx->d_img, n, d_max);
        else if (dtype == EUCALC_I16) maxabs_kernel<<<g, 256, 0, st>>>((const int16_t *)cx->d_img, n, d_max);
        else maxabs_kernel<<<g, 256, 0, st>>>((const int32_t *)cx->d_img, n, d_max);
        count_launch();
        e = cudaGetLastError();
    }
    unsigned long long hmax = 0;
    if (e == cudaSuccess) e = cudaMemcpyAsync(&hmax, d_max, sizeof(hmax), cudaMemcpyDeviceToHost, st);
    if (d_max) cudaFreeAsync(d_max, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) {
        cudaFreeAsync(cx->d_img, st);
        delete cx;
        return cuda_fail(e, "build_complex");
    }
    cx->max_abs_w = (int64_t)hmax;
    cx->owner_stream = st;
    *out = cx;
    return EUCALC_OK;
}

eucalc_status eucalc_destroy_complex(eucalc_complex *cx) {
    if (!cx) return fail(EUCALC_E_STATE, "NULL handle");
    // stream-ordered release on the stream the handle was built on (no device
    // sync), after the work other streams enqueued on it
    cx->users.join(cx->owner_stream);
    if (cx->d_img) cudaFreeAsync(cx->d_img, cx->owner_stream);
    delete cx;
    return EUCALC_OK;
}

eucalc_status eucalc_critical_points(const eucalc_complex *cx, void *stream, eucalc_critical **out) {
    if (!out) return fail(EUCALC_E_ARG, "out is NULL");
    *out = nullptr;
    if (!cx || !cx->d_img) return fail(EUCALC_E_STATE, "invalid complex");
    cudaStream_t st = (cudaStream_t)stream;
    const_cast<eucalc_complex *>(cx)->users.note(st, cx->owner_stream);
    eucalc_critical *cr = new (std::nothrow) eucalc_critical();
    if (!cr) return fail(EUCALC_E_NOMEM, "host alloc");
    const int n = cx->ndim;
    cr->cx = cx;
    cr->owner_stream = st;
    cr->Q = 1 << (n - 1);
    // |Delta^-| <= 2^n max|w| must fit the record's int16 halves, J = a - b is formed in int32
    cr->wide = ((int64_t(1) << n) * cx->max_abs_w) > 32767;
    cr->vcap = cx->nvert;
    const size_t rsz = cr->wide ? sizeof(Rec32) : sizeof(Rec16);
    const int64_t nlist = cx->batch * cr->Q;
    const int64_t nstats = cx->batch * (1 << n) * 2 + 2 * nlist;
    // tiles (K2's culling unit and K1's offset granularity): boxes of TX x TY x TZ
    // vertices, W pencils (warps) each (k1_critical.cu)
    int TX, TY, TZ, W;
    k1_geometry(n, cx->M, cx->dtype, cx->construction, &TX, &TY, &TZ, &W);
    const int MX = (int)cx->M[n - 1], MY = (int)cx->M[n - 2], MZ = n == 3 ? (int)cx->M[0] : 1;
    cr->TX = TX;
    cr->TY = TY;
    cr->TZ = TZ;
    cr->tiles_x = (MX + TX - 1) / TX;
    cr->tiles_y = (MY + TY - 1) / TY;
    cr->tiles_z = n == 3 ? (MZ + TZ - 1) / TZ : 1;
    cr->ntiles = cr->tiles_x * cr->tiles_y * cr->tiles_z;
    const int64_t ncnt = nlist * (int64_t)cr->ntiles * W;
    const int64_t nflags = k1_scan_chunks(nlist, cr->ntiles, W);
    // K1 scratch: (tile, warp) counts, scan flags, scan ticket (one allocation, zeroed)
    const size_t cnt_bytes = ((sizeof(int32_t) * ncnt + 15) / 16) * 16;
    const size_t scratch_bytes = cnt_bytes + sizeof(unsigned long long) * nflags + 16;
    int32_t *cnt = nullptr;
    cudaError_t e = cudaMallocAsync(&cr->d_rec, rsz * nlist * cr->vcap, st);
    if (e == cudaSuccess) e = cudaMallocAsync(&cr->d_count, sizeof(int32_t) * nlist, st);
    if (e == cudaSuccess) e = cudaMallocAsync(&cr->d_tile_off, sizeof(int32_t) * nlist * (cr->ntiles + 1), st);
    if (e == cudaSuccess) e = cudaMallocAsync(&cr->d_stats, sizeof(int64_t) * nstats, st);
    // records in fixed-capacity (tile, warp) regions before the copy to the lists
    const int cap_r = TX * (n == 3 ? TZ : TY / W);
    const int64_t scap = (int64_t)cr->ntiles * W * cap_r;
    const bool direct = (int64_t)cr->ntiles * W == 1;
    void *rscratch = nullptr;
    if (e == cudaSuccess) e = cudaMallocAsync(&cnt, scratch_bytes, st);
    if (e == cudaSuccess && !direct) e = cudaMallocAsync(&rscratch, rsz * nlist * scap, st);
    if (e == cudaSuccess) e = cudaMemsetAsync(cr->d_stats, 0, sizeof(int64_t) * nstats, st);
    if (e == cudaSuccess) e = cudaMemsetAsync(cnt, 0, scratch_bytes, st);
    if (e == cudaSuccess) {
        K1Args a = k1_args(cr);
        a.cnt = cnt;
        a.flags = (unsigned long long *)((unsigned char *)cnt + cnt_bytes);
        a.ticket = (unsigned int *)(a.flags + nflags);
        a.scratch = rscratch;
        a.scap = scap;
        a.cap_r = cap_r;
        a.direct = direct;
        {
            ProfScope ps("k1_critical", st);
            e = launch_k1(a, st);
        }
        // asynchronous read-back of the list lengths and |Delta^-| statistics into
        // pinned memory; sync_counts() later waits on this event only
        cr->pinned_stats_off = ((sizeof(int32_t) * nlist + 15) / 16) * 16;
        const size_t flag_off = ((cr->pinned_stats_off + sizeof(int64_t) * nstats + 15) / 16) * 16;
        const size_t need = flag_off + 16;
        cr->pinned = pinned_get(need, &cr->pinned_bytes);
        if (e == cudaSuccess && !cr->pinned) e = cudaErrorMemoryAllocation;
        unsigned *dflag = nullptr;
        if (e == cudaSuccess) {
            *(volatile unsigned *)((unsigned char *)cr->pinned + flag_off) = 0u;
            if (cudaHostGetDevicePointer((void **)&dflag, (unsigned char *)cr->pinned + flag_off, 0) != cudaSuccess) {
                cudaGetLastError();
                dflag = nullptr;
            }
        }
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&cr->k1_done, cudaEventDisableTiming);
        if (e == cudaSuccess)
            e = cudaMemcpyAsync(cr->pinned, cr->d_count, sizeof(int32_t) * nlist, cudaMemcpyDeviceToHost, st);
        if (e == cudaSuccess)
            e = cudaMemcpyAsync((unsigned char *)cr->pinned + cr->pinned_stats_off, cr->d_stats,
                                sizeof(int64_t) * nstats, cudaMemcpyDeviceToHost, st);
        if (e == cudaSuccess && dflag) {
            k1_signal<<<1, 1, 0, st>>>(dflag, 1u);
            count_launch();
            e = cudaGetLastError();
            if (e == cudaSuccess) cr->pinned_flag_off = flag_off;
        }
        if (e == cudaSuccess) e = cudaEventRecord(cr->k1_done, st);
    }
    if (cnt) cudaFreeAsync(cnt, st);
    if (rscratch) cudaFreeAsync(rscratch, st);
    if (e != cudaSuccess) {
        if (cr->d_rec) cudaFreeAsync(cr->d_rec, st);
        if (cr->d_count) cudaFreeAsync(cr->d_count, st);
        if (cr->d_tile_off) cudaFreeAsync(cr->d_tile_off, st);
        if (cr->d_stats) cudaFreeAsync(cr->d_stats, st);
        if (cr->k1_done) cudaEventDestroy(cr->k1_done);
        cudaStreamSynchronize(st);
        pinned_put(cr->pinned, cr->pinned_bytes);
        delete cr;
        return cuda_fail(e, "critical_points");
    }
    *out = cr;
    return EUCALC_OK;
}

eucalc_status eucalc_destroy_critical(eucalc_critical *cr) {
    if (!cr) return fail(EUCALC_E_STATE, "NULL handle");
    cr->users.join(cr->owner_stream);
    cudaFreeAsync(cr->d_rec, cr->owner_stream);
    cudaFreeAsync(cr->d_count, cr->owner_stream);
    cudaFreeAsync(cr->d_tile_off, cr->owner_stream);
    cudaFreeAsync(cr->d_stats, cr->owner_stream);
    if (cr->k1_done) {
        cudaEventSynchronize(cr->k1_done);  // the read-back into `pinned` has landed
        cudaEventDestroy(cr->k1_done);
    }
    pinned_put(cr->pinned, cr->pinned_bytes);
    delete[] cr->h_count;
    delete[] cr->h_stats;
    delete cr;
    return EUCALC_OK;
}

eucalc_status eucalc_critical_counts(const eucalc_critical *ccr, int64_t *h_counts, void *stream) {
    if (!ccr || !h_counts) return fail(EUCALC_E_ARG, "NULL argument");
    eucalc_critical *cr = const_cast<eucalc_critical *>(ccr);
    cudaStream_t st = (cudaStream_t)stream;
    eucalc_status s = sync_counts(cr, st);
    if (s != EUCALC_OK) return s;
    const size_t nb = sizeof(int64_t) * cr->cx->batch * (1 << cr->cx->ndim) * 2;
    std::lock_guard<std::mutex> lk(cr->mu);
    if (!cr->have_orthant_counts) {
        // N^-, N^ord per orthant: the K1 stencil once more, counting only
        cr->users.note(st, cr->owner_stream);
        CK(launch_k1_stats(k1_args(cr), st));
        CK(cudaMemcpyAsync(cr->h_stats, cr->d_stats, nb, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        cr->have_orthant_counts = true;
    }
    memcpy(h_counts, cr->h_stats, nb);
    return EUCALC_OK;
}

eucalc_status eucalc_critical_list_lengths(const eucalc_critical *ccr, int64_t *h_len, void *stream) {
    if (!ccr || !h_len) return fail(EUCALC_E_ARG, "NULL argument");
    eucalc_critical *cr = const_cast<eucalc_critical *>(ccr);
    eucalc_status s = sync_counts(cr, (cudaStream_t)stream);
    if (s != EUCALC_OK) return s;
    memcpy(h_len, cr->h_count, sizeof(int64_t) * cr->cx->batch * cr->Q);
    return EUCALC_OK;
}

eucalc_status eucalc_critical_export(const eucalc_critical *ccr, int64_t image, int orthant, int64_t *vertex,
                                     int32_t *dminus, int32_t *jump, int64_t cap, int64_t *n_out, void *stream) {
    if (!ccr || !n_out) return fail(EUCALC_E_ARG, "NULL argument");
    eucalc_critical *cr = const_cast<eucalc_critical *>(ccr);
    const Complex *cx = cr->cx;
    const int n = cx->ndim, full = (1 << n) - 1;
    if (image < 0 || image >= cx->batch || orthant < 0 || orthant > full) return fail(EUCALC_E_ARG, "bad image/orthant");
    cudaStream_t st = (cudaStream_t)stream;
    eucalc_status s = sync_counts(cr, st);
    if (s != EUCALC_OK) return s;
    const bool rep = ((orthant >> (n - 1)) & 1) == 0;
    const int q = rep ? orthant : (orthant ^ full);
    const int64_t len = cr->h_count[image * cr->Q + q];
    *n_out = len;
    if (cap < len) return fail(EUCALC_E_CAPACITY, "export capacity");
    const size_t rsz = cr->wide ? sizeof(Rec32) : sizeof(Rec16);
    std::vector<unsigned char> raw(rsz * len);
    if (len) {
        CK(cudaMemcpyAsync(raw.data(), (const unsigned char *)cr->d_rec + rsz * (image * cr->Q + q) * cr->vcap,
                           rsz * len, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
    }
    struct Row { int64_t v; int32_t dm, j; };
    std::vector<Row> rows(len);
    for (int64_t i = 0; i < len; ++i) {
        uint32_t c;
        int32_t a, b;
        if (cr->wide) {
            const Rec32 *r = (const Rec32 *)raw.data() + i;
            c = r->c; a = r->a; b = r->b;
        } else {
            const Rec16 *r = (const Rec16 *)raw.data() + i;
            c = r->c; a = r->a; b = r->b;
        }
        int64_t vid = 0;
        for (int k = 0; k < n; ++k) vid = vid * cx->M[k] + ((c >> cx->sh[k]) & cx->msk[k]);
        const int32_t dm = rep ? a : b, other = rep ? b : a;
        rows[i] = Row{vid, dm, dm - other};
    }
    std::sort(rows.begin(), rows.end(), [](const Row &x, const Row &y) { return x.v < y.v; });
    std::vector<int64_t> hv(len);
    std::vector<int32_t> hd(len), hj(len);
    for (int64_t i = 0; i < len; ++i) { hv[i] = rows[i].v; hd[i] = rows[i].dm; hj[i] = rows[i].j; }
    auto put = [&](void *dst, const void *src, size_t bytes) -> cudaError_t {
        if (!dst || !bytes) return cudaSuccess;
        if (is_device_ptr(dst)) return cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, st);
        memcpy(dst, src, bytes);
        return cudaSuccess;
    };
    CK(put(vertex, hv.data(), sizeof(int64_t) * len));
    CK(put(dminus, hd.data(), sizeof(int32_t) * len));
    CK(put(jump, hj.data(), sizeof(int32_t) * len));
    CK(cudaStreamSynchronize(st));
    return EUCALC_OK;
}

eucalc_status eucalc_output_bound(const eucalc_critical *ccr, const int32_t *dirs, int64_t D, int64_t *bound_ect,
                                  int64_t *bound_ordinary, void *stream) {
    if (!ccr) return fail(EUCALC_E_STATE, "NULL handle");
    eucalc_critical *cr = const_cast<eucalc_critical *>(ccr);
    std::shared_ptr<PlanEntry> pe;
    eucalc_status s = get_plan(cr->cx, dirs, D, (cudaStream_t)stream, pe);
    if (s != EUCALC_OK) return s;
    int64_t bnd = 0;
    s = bounds(cr, pe->p, (cudaStream_t)stream, bnd);
    if (s != EUCALC_OK) return s;
    if (bound_ect) *bound_ect = bnd;
    if (bound_ordinary) *bound_ordinary = bnd;
    return EUCALC_OK;
}

eucalc_status eucalc_output_bound_upper(const eucalc_complex *cx, const int32_t *dirs, int64_t D, int64_t *bound,
                                        void *stream) {
    if (!cx || !bound) return fail(EUCALC_E_ARG, "NULL argument");
    std::shared_ptr<PlanEntry> pe;
    eucalc_status s = get_plan(cx, dirs, D, (cudaStream_t)stream, pe);
    if (s != EUCALC_OK) return s;
    int64_t b = 0;
    for (const DirInfo &di : pe->p.info) b += std::min<int64_t>(cx->nvert, di.R);
    *bound = b * cx->batch;
    return EUCALC_OK;
}

}  // extern "C"

namespace {
constexpr int64_t kFusedTabMax = int64_t(1) << 24;  // kbar entries of the fused HT table (128 MB)

struct HtReq {
    int kernel, precision;
    double param;
    void *out;
};

eucalc_status transforms_impl(const eucalc_critical *ccr, const int32_t *dirs, int64_t D, eucalc_steps *ect,
                              eucalc_steps *ordinary, eucalc_steps *classical, const HtReq *ht, int64_t *required_out,
                              void *stream);

// The library's device-to-host copy stream of the current device (non-blocking).
cudaStream_t copy_stream() {
    static std::mutex mu;
    static cudaStream_t s[64] = {};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return nullptr;
    std::lock_guard<std::mutex> lk(mu);
    if (!s[dev] && cudaStreamCreateWithFlags(&s[dev], cudaStreamNonBlocking) != cudaSuccess) {
        cudaGetLastError();
        s[dev] = nullptr;
    }
    return s[dev];
}

// Host outputs in chunks of images (and, when every chunk is one image, of
// direction ranges of that image): the transforms of every chunk are enqueued on
// `st` into device scratch (a view of the critical handle restricted to the
// chunk's images, the chunk's directions, its own CSR), and each chunk's results
// are copied back on the copy stream while the next chunks compute; offsets are
// shifted to the global CSR on the host. Capacities and ranges were checked for
// the whole call by the caller.
eucalc_status transforms_host_chunked(eucalc_critical *cr, const int32_t *dirs, int64_t D, eucalc_steps *const outs[3],
                                      bool cls_alias, int eb, const HtReq *ht, int64_t nch, int64_t ndch,
                                      cudaStream_t st) {
    const Complex *cx = cr->cx;
    const int64_t B = cx->batch;
    const size_t esz = (size_t)eb, rsz = cr->wide ? sizeof(Rec32) : sizeof(Rec16);
    const size_t ht_osz = ht && ht->precision == EUCALC_F32 ? 4 : 8;
    cudaStream_t cs = copy_stream();
    if (!cs) return fail(EUCALC_E_CUDA, "copy stream");
    eucalc_status s = EUCALC_OK;
    // single-image chunks are cut further into `ndch` direction ranges (the CSR is
    // image-major, so (image, direction range) chunks in that order stay contiguous)
    if (nch < B) ndch = 1;
    ndch = std::max<int64_t>(1, std::min<int64_t>(ndch, D));
    struct Chunk {
        eucalc_complex vcx;
        eucalc_critical vcr;
        int64_t b0 = 0, nb = 0, d0 = 0, nd = 0;
        StepsOut dv[3] = {};
        void *dht = nullptr;
        cudaEvent_t ev = nullptr;
        std::vector<void *> mem;
    };
    std::vector<std::unique_ptr<Chunk>> chunks;
    auto release = [&]() {
        for (auto &c : chunks) {
            for (void *q : c->mem) cudaFreeAsync(q, cs);
            if (c->ev) cudaEventDestroy(c->ev);
        }
    };
    cudaError_t e = cudaSuccess;
    for (int64_t cc = 0; cc < nch * ndch && s == EUCALC_OK && e == cudaSuccess; ++cc) {
        const int64_t c = cc / ndch, dc = cc % ndch;
        auto ch = std::make_unique<Chunk>();
        ch->b0 = B * c / nch;
        ch->nb = B * (c + 1) / nch - ch->b0;
        ch->d0 = D * dc / ndch;
        ch->nd = D * (dc + 1) / ndch - ch->d0;
        const int32_t *cdirs = dirs + ch->d0 * cx->ndim;
        std::shared_ptr<PlanEntry> pe;
        s = get_plan(cx, cdirs, ch->nd, st, pe);
        if (s != EUCALC_OK) break;
        Complex &v = ch->vcx;
        v.ndim = cx->ndim;
        v.dtype = cx->dtype;
        v.construction = cx->construction;
        v.batch = ch->nb;
        std::copy(cx->m, cx->m + kMaxN, v.m);
        std::copy(cx->M, cx->M + kMaxN, v.M);
        v.npix = cx->npix;
        v.nvert = cx->nvert;
        v.d_img = (unsigned char *)cx->d_img + ch->b0 * cx->npix * (cx->dtype == EUCALC_U8 ? 1 : cx->dtype == EUCALC_I16 ? 2 : 4);
        v.max_abs_w = cx->max_abs_w;
        std::copy(cx->sh, cx->sh + kMaxN, v.sh);
        std::copy(cx->msk, cx->msk + kMaxN, v.msk);
        v.aligned = cx->aligned;
        v.L = cx->L;
        std::copy(cx->scale, cx->scale + kMaxN, v.scale);
        v.owner_stream = st;
        Critical &r = ch->vcr;
        r.cx = &ch->vcx;
        r.Q = cr->Q;
        r.wide = cr->wide;
        r.vcap = cr->vcap;
        r.d_rec = (unsigned char *)cr->d_rec + (size_t)(ch->b0 * cr->Q) * (size_t)cr->vcap * rsz;
        r.d_count = cr->d_count + ch->b0 * cr->Q;
        r.d_tile_off = cr->d_tile_off + ch->b0 * cr->Q * (int64_t)(cr->ntiles + 1);
        r.TX = cr->TX;
        r.TY = cr->TY;
        r.TZ = cr->TZ;
        r.tiles_x = cr->tiles_x;
        r.tiles_y = cr->tiles_y;
        r.tiles_z = cr->tiles_z;
        r.ntiles = cr->ntiles;
        r.have_host = true;
        r.h_count = cr->h_count + ch->b0 * cr->Q;
        r.max_count = cr->max_count;
        r.max_abs_sum = cr->max_abs_sum;
        r.max_rec = cr->max_rec;
        r.owner_stream = st;
        int64_t bnd = 0;
        s = bounds(&ch->vcr, pe->p, st, bnd);
        if (s != EUCALC_OK) break;
        const int64_t Sc = ch->nb * ch->nd;
        auto dalloc = [&](size_t bytes) -> void * {
            void *q = nullptr;
            if (cudaMallocAsync(&q, std::max<size_t>(bytes, 1), st) != cudaSuccess) return nullptr;
            ch->mem.push_back(q);
            return q;
        };
        eucalc_steps ds[3] = {};
        eucalc_steps *dsp[3] = {nullptr, nullptr, nullptr};
        for (int i = 0; i < 3 && e == cudaSuccess; ++i) {
            if (!outs[i]) continue;
            ch->dv[i].off = (int64_t *)dalloc(sizeof(int64_t) * (Sc + 1));
            ch->dv[i].v = dalloc(esz * std::max<int64_t>(bnd, 1));
            ch->dv[i].h = (i == 2 && cls_alias) ? ch->dv[0].h : dalloc(esz * std::max<int64_t>(bnd, 1));
            if (!ch->dv[i].off || !ch->dv[i].v || !ch->dv[i].h) e = cudaErrorMemoryAllocation;
            ds[i] = eucalc_steps{ch->dv[i].off, ch->dv[i].h, ch->dv[i].v, std::max<int64_t>(bnd, 1), eb, 0};
            dsp[i] = &ds[i];
        }
        HtReq hc{};
        if (ht && e == cudaSuccess) {
            hc = *ht;
            ch->dht = dalloc(ht_osz * std::max<int64_t>(Sc, 1));
            hc.out = ch->dht;
            if (!ch->dht) e = cudaErrorMemoryAllocation;
        }
        if (e != cudaSuccess) break;
        s = transforms_impl(&ch->vcr, cdirs, ch->nd, dsp[0], dsp[1], dsp[2], ht ? &hc : nullptr, nullptr, st);
        if (s != EUCALC_OK) break;
        e = cudaEventCreateWithFlags(&ch->ev, cudaEventDisableTiming);
        if (e == cudaSuccess) e = cudaEventRecord(ch->ev, st);
        chunks.push_back(std::move(ch));
    }
    if (s != EUCALC_OK || e != cudaSuccess) {
        cudaStreamSynchronize(st);
        release();
        cudaStreamSynchronize(cs);
        return s != EUCALC_OK ? s : cuda_fail(e, "chunked transforms");
    }
    // copy back chunk by chunk (each after its own event) while later chunks compute
    int64_t base[3] = {0, 0, 0};
    for (auto &ch : chunks) {
        const int64_t Sc = ch->nb * ch->nd, s0 = ch->b0 * D + ch->d0;
        if (e == cudaSuccess) e = cudaStreamWaitEvent(cs, ch->ev, 0);
        for (int i = 0; i < 3 && e == cudaSuccess; ++i)
            if (outs[i]) e = cudaMemcpyAsync(outs[i]->offsets + s0, ch->dv[i].off, sizeof(int64_t) * (Sc + 1),
                                             cudaMemcpyDeviceToHost, cs);
        if (e == cudaSuccess) e = cudaStreamSynchronize(cs);
        for (int i = 0; i < 3 && e == cudaSuccess; ++i) {
            eucalc_steps *o = outs[i];
            if (!o) continue;
            const int64_t n = o->offsets[s0 + Sc];
            if (n > 0) {
                e = cudaMemcpyAsync((unsigned char *)o->value + (size_t)base[i] * esz, ch->dv[i].v, esz * (size_t)n,
                                    cudaMemcpyDeviceToHost, cs);
                if (e == cudaSuccess && o->height && !(i == 2 && cls_alias))
                    e = cudaMemcpyAsync((unsigned char *)o->height + (size_t)base[i] * esz, ch->dv[i].h,
                                        esz * (size_t)n, cudaMemcpyDeviceToHost, cs);
            }
            for (int64_t k = 0; k <= Sc; ++k) o->offsets[s0 + k] += base[i];
            base[i] += n;
        }
        if (e == cudaSuccess && ht)
            e = cudaMemcpyAsync((unsigned char *)ht->out + (size_t)s0 * ht_osz, ch->dht, ht_osz * (size_t)Sc,
                                cudaMemcpyDeviceToHost, cs);
    }
    release();
    const cudaError_t e2 = cudaStreamSynchronize(cs);
    if (e == cudaSuccess) e = e2;
    if (e != cudaSuccess) return cuda_fail(e, "chunked transforms copy-back");
    return EUCALC_OK;
}

eucalc_status transforms_impl(const eucalc_critical *ccr, const int32_t *dirs, int64_t D, eucalc_steps *ect,
                              eucalc_steps *ordinary, eucalc_steps *classical, const HtReq *ht, int64_t *required_out,
                              void *stream) {
    HostTrace tr("transforms");
    if (!ccr) return fail(EUCALC_E_STATE, "NULL handle");
    if (ht) {
        if (ht->kernel < EUCALC_K_GAUSS || ht->kernel > EUCALC_K_EXP) return fail(EUCALC_E_ARG, "bad kernel");
        if (ht->precision != EUCALC_F32 && ht->precision != EUCALC_F64) return fail(EUCALC_E_ARG, "bad precision");
        if ((ht->kernel == EUCALC_K_GAUSS || ht->kernel == EUCALC_K_COS) && !(ht->param > 0))
            return fail(EUCALC_E_ARG, "param must be > 0");
        if (D > 0 && !ht->out) return fail(EUCALC_E_ARG, "ht_out is NULL");
        if (!ordinary) return fail(EUCALC_E_ARG, "the fused HT needs the ordinary stream");
    }
    eucalc_critical *cr = const_cast<eucalc_critical *>(ccr);
    const Complex *cx = cr->cx;
    cudaStream_t st = (cudaStream_t)stream;
    cr->users.note(st, cr->owner_stream);
    std::shared_ptr<PlanEntry> pe;
    eucalc_status s = get_plan(cx, dirs, D, st, pe);
    if (s != EUCALC_OK) return s;
    tr.mark("plan");
    const DirPlan &p = pe->p;
    if (ht) {
        // the fused HT tabulates kbar over the directions' whole u range (8 B per
        // u); beyond kFusedTabMax entries (unequal extents make L, hence U, large)
        // the transforms run unfused and the HT comes from K3, which evaluates
        // kbar per term when its table does not apply (same tolerance, E18).
        // EUCALC_FUSED_TAB_MAX overrides the limit (test hook).
        int64_t tab_max = kFusedTabMax;
        if (const char *v = getenv("EUCALC_FUSED_TAB_MAX")) tab_max = std::max<int64_t>(1, atoll(v));
        if (p.U1 - p.U0 + 1 > tab_max) {
            s = transforms_impl(ccr, dirs, D, ect, ordinary, classical, nullptr, required_out, stream);
            if (s != EUCALC_OK) return s;
            return eucalc_hybrid_ex(ccr, dirs, D, ht->kernel, ht->param, ht->precision, EUCALC_HT_AUTO, ht->out,
                                    stream);
        }
    }
    // Output bound: the tight one (sum over (image, direction) of min(list length,
    // R), O(batch * Q * log D) on the host, ~60 us at config 2's 2048 images) only
    // when the no-K1 upper bound (sum of min(vertices, R), O(D)) is not already
    // covered by every capacity, or host outputs need scratch sized by it.
    s = sync_counts(cr, st);
    if (s != EUCALC_OK) return s;
    tr.mark("k1 wait");
    eucalc_steps *outs[3] = {ect, ordinary, classical};
    bool host_out = false;
    for (eucalc_steps *o : outs)
        if (o && o->value && !is_device_ptr(o->value)) host_out = true;
    int64_t bnd = 0;
    {
        int64_t ub = 0;
        for (const DirInfo &di : p.info) ub += std::min<int64_t>(cx->nvert, di.R);
        ub *= cx->batch;
        bool covered = !host_out && ub < (int64_t(1) << 31);
        for (eucalc_steps *o : outs)
            if (o && o->capacity < ub) covered = false;
        if (covered) {
            bnd = ub;
        } else {
            s = bounds(cr, p, st, bnd);
            if (s != EUCALC_OK) return s;
        }
    }
    tr.mark("bound");
    if (required_out) *required_out = bnd;
    int eb = 0;
    for (eucalc_steps *o : outs) {
        if (!o) continue;
        if (!o->offsets || (!o->height && o != classical) || !o->value) return fail(EUCALC_E_ARG, "NULL output array");
        if (o->elem_bytes != 2 && o->elem_bytes != 4 && o->elem_bytes != 8) return fail(EUCALC_E_ARG, "elem_bytes must be 2, 4 or 8");
        if (eb && o->elem_bytes != eb) return fail(EUCALC_E_ARG, "all outputs must share elem_bytes");
        eb = o->elem_bytes;
        if (o->capacity < bnd) return fail(EUCALC_E_CAPACITY, "capacity " + std::to_string(o->capacity) + " < required bound " + std::to_string(bnd));
    }
    if (!eb) return EUCALC_OK;  // nothing requested
    // value bounds: every bin sum, ECT and Radon value is bounded by the list's sum |a|+|b|
    if (cr->max_abs_sum >= (int64_t(1) << 31)) return fail(EUCALC_E_RANGE, "total |weight| of a critical list exceeds 2^31");
    if (bnd >= (int64_t(1) << 31)) return fail(EUCALC_E_RANGE, "more than 2^31 output entries in one call");
    if (eb == 2) {
        bool fits = cr->max_abs_sum < 32768;
        for (const DirInfo &di : p.info) fits = fits && di.hlo >= -32768 && (int64_t)di.hlo + di.R - 1 <= 32767;
        if (!fits) return fail(EUCALC_E_RANGE, "heights or values do not fit int16 (elem_bytes 2)");
    }
    const int64_t S = cx->batch * D;
    if (S == 0) return EUCALC_OK;
    // the warp-regime loops step int32 segment indices by the grid's warp count
    // (< 2^24): keep s + step below 2^31
    if (S > INT32_MAX - (int64_t(1) << 24))
        return fail(EUCALC_E_RANGE, "more than 2^31 - 2^24 (image, direction) segments in one call");
    const bool cls_alias = classical && ect && (classical->height == ect->height || !classical->height);
    if (classical && !classical->height && !ect) return fail(EUCALC_E_ARG, "classical height is NULL");
    // host outputs of several images: chunked, copy-back overlapped with the next chunks
    // (a chunk of one image is cut further into direction ranges when the call is large:
    // more than 2^22 output entries per range, so small calls keep one launch per image)
    if (host_out) {
        const char *ev = getenv("EUCALC_HOST_CHUNKS"), *dv = getenv("EUCALC_HOST_DIR_CHUNKS");
        const int64_t nch = std::min<int64_t>(cx->batch, ev ? std::max(1, atoi(ev)) : 4);
        int64_t ndch = 1;
        if (nch == cx->batch) {
            const int64_t per_image = bnd / std::max<int64_t>(1, cx->batch);
            ndch = dv ? std::max(1, atoi(dv)) : (per_image >> 22) ? 2 : 1;  // measured: 2 best (config 4), more ranges leave SMs idle
            ndch = std::max<int64_t>(1, std::min<int64_t>(ndch, D));
        }
        if (nch * ndch >= 2) {
            bool all_host = true;  // every output on the host (mixed placements take the plain path)
            for (eucalc_steps *o : outs)
                if (o && is_device_ptr(o->value)) all_host = false;
            if (ht && is_device_ptr(ht->out)) all_host = false;
            if (all_host) return transforms_host_chunked(cr, dirs, D, outs, cls_alias, eb, ht, nch, ndch, st);
        }
    }
    // host outputs -> device scratch (sized by the tight bound)
    const size_t esz = (size_t)eb;
    std::vector<void *> scratch;
    auto dalloc = [&](size_t bytes) -> void * {
        void *q = nullptr;
        if (cudaMallocAsync(&q, bytes, st) != cudaSuccess) return nullptr;
        scratch.push_back(q);
        return q;
    };
    auto free_scratch = [&]() { for (void *q : scratch) cudaFreeAsync(q, st); };
    K2Args a{};
    StepsOut dev[3] = {};
    for (int i = 0; i < 3; ++i) {
        eucalc_steps *o = outs[i];
        if (!o) continue;
        if (host_out) {
            dev[i].off = (int64_t *)dalloc(sizeof(int64_t) * (S + 1));
            dev[i].v = dalloc(esz * std::max<int64_t>(bnd, 1));
            dev[i].h = (i == 2 && cls_alias) ? dev[0].h : dalloc(esz * std::max<int64_t>(bnd, 1));
            if (!dev[i].off || !dev[i].v || !dev[i].h) {
                free_scratch();
                return fail(EUCALC_E_NOMEM, "device scratch for host outputs");
            }
        } else {
            dev[i].off = o->offsets;
            dev[i].h = (i == 2 && cls_alias) ? nullptr : o->height;
            dev[i].v = o->value;
        }
    }
    const DirInfo *d_info = pe->d_info;
    // warp regime, lists of <= 32 records: k2w_count keeps the merged runs (16-bit
    // fields: every bin index, value and running sum must fit) so that k2w_emit
    // need not sort them again
    int64_t min_count = INT64_MAX;
    for (int64_t i = 0; i < cx->batch * cr->Q; ++i) min_count = std::min(min_count, cr->h_count[i]);
    int sparse_max = 32;  // EUCALC_K2_SPARSE_MAX (0..32) overrides, for measurements
    if (const char *v = getenv("EUCALC_K2_SPARSE_MAX")) sparse_max = std::max(0, std::min(32, atoi(v)));
    if (p.R_max >= (1 << 25)) sparse_max = 0;  // the register sort keys are bin << 5 | lane
    const bool slab_ok = min_count <= sparse_max && p.R_max <= 32767 && cr->max_abs_sum < 32768 && cr->max_count <= 32768;
    // fused HT: the kbar table over the directions' u range, and the output
    const int64_t U = p.U1 - p.U0 + 1;
    const bool ht_host = ht && !is_device_ptr(ht->out);
    const size_t ht_osz = ht && ht->precision == EUCALC_F32 ? 4 : 8;
    // flags + ticket are adjacent (one memset); then counts, slab, table, HT staging
    std::vector<void *> ar;
    if (!arena_take(st, {sizeof(unsigned long long) * S + sizeof(unsigned int) * 4, sizeof(int) * 2 * S,
                         slab_ok ? sizeof(uint2) * 33 * S : 0, ht ? 8 * (size_t)U : 0,
                         ht_host ? ht_osz * S : 0},
                    ar)) {
        free_scratch();
        return fail(EUCALC_E_NOMEM, "scratch");
    }
    tr.mark("checks+arena");
    unsigned long long *flags = (unsigned long long *)ar[0];
    unsigned int *ticket = (unsigned int *)(flags + S);
    int *cnts = (int *)ar[1];
    uint2 *slab = (uint2 *)ar[2];
    double *d_tab = (double *)ar[3];
    void *d_ht = ht ? (ht_host ? ar[4] : ht->out) : nullptr;
    cudaError_t e = cudaMemsetAsync(flags, 0, sizeof(unsigned long long) * S + sizeof(unsigned int) * 4, st);
    if (e == cudaSuccess && ht)
        e = launch_k3_table_only(ht->kernel, ht->param, cx->L, p.U0, U, d_tab, nullptr, st);
    if (e == cudaSuccess) {
        a.ht_tab = d_tab;
        a.ht_U0 = p.U0;
        a.ht_U = U;
        a.L = cx->L;
        a.csum = pe->d_csum;
        a.ht_scale = ht ? k3_scale(ht->kernel, ht->param) : 0.0;
        a.ht_prec = ht ? ht->precision : 0;
        a.ht_out = d_ht;
        a.rec = cr->d_rec;
        a.wide = cr->wide;
        a.vcap = cr->vcap;
        a.count = cr->d_count;
        a.Q = cr->Q;
        a.ndim = cx->ndim;
        for (int k = 0; k < cx->ndim; ++k) {
            a.sh[k] = cx->sh[k];
            a.msk[k] = cx->msk[k];
        }
        a.dirs = d_info;
        a.tile_off = cr->d_tile_off;
        a.ntiles = cr->ntiles;
        a.tiles_x = cr->tiles_x;
        a.tiles_y = cr->tiles_y;
        a.TX = cr->TX;
        a.TY = cr->TY;
        a.TZ = cr->TZ;
        for (int k = 0; k < cx->ndim; ++k) a.M[k] = (int)cx->M[k];
        a.D = D;
        a.batch = cx->batch;
        a.R_max = p.R_max;
        a.max_count = cr->max_count;
        a.elem_bytes = eb;
        a.pack16 = bin_sum_bound(cr) < 32768;
        a.dp = p.dp;
        a.do_ect = ect != nullptr;
        a.do_ord = ordinary != nullptr;
        a.do_cls = classical != nullptr;
        a.cls_alias = cls_alias;
        a.ect = dev[0];
        a.ord = dev[1];
        a.cls = dev[2];
        a.out_cap = INT64_MAX;  // device checks: the smallest capacity of the requested outputs
        for (int i = 0; i < 3; ++i)
            if (outs[i]) a.out_cap = std::min<int64_t>(a.out_cap, host_out ? std::max<int64_t>(bnd, 1) : outs[i]->capacity);
        if (getenv("EUCALC_DCHECK_INJECT")) a.out_cap = 1;  // test hook: the checked library must trap
        a.flags = flags;
        a.ticket = ticket;
        a.cnt_c = cnts;
        a.cnt_o = cnts + S;
        a.slab = slab;
        a.sparse_max = sparse_max;
        a.sum16 = cr->max_abs_sum < 32768;
        a.max_rec = cr->max_rec;
        a.max_abs_sum = cr->max_abs_sum;
        a.no_chk = getenv("EUCALC_K2_NO_CHK") != nullptr;
        {
            int k = 14;  // test hook: a narrower checked range forces the split-bin restart
            if (const char *v = getenv("EUCALC_K2_CHK_BITS")) k = std::max(1, std::min(14, atoi(v)));
            a.chk_bias = (1u << k) * 0x10001u;
            a.chk_mask = ((0xffffu << (k + 1)) & 0xffffu) * 0x10001u;
        }
        tr.mark("memset+table+args");
        // block regime, unit path: several directions per pass over a list, every
        // segment staged (fixed slot of R_d entries per stream) — needs byte-aligned
        // coordinates, 8-byte records, single-window split fallback, checked packing
        bool unit = false;
        {
            const char *ev = getenv("EUCALC_K2_UNIT");
            const bool want = !(ev && ev[0] == '0');
            if (want && !cr->wide && p.dp == 3 && k2_block_regime(a) && a.max_rec < 16384 &&
                !a.no_chk && p.R_max <= k2_split_window()) {
                s = plan_units(*pe);
                if (s != EUCALC_OK) {
                    free_scratch();
                    return s;
                }
                const size_t sb = 6 * (size_t)cx->batch * (size_t)pe->stage_img * esz;
                if (pe->nunits > 0 && sb <= (size_t(4) << 30)) {
                    a.stage = dalloc(sb);
                    if (a.stage) {
                        a.units = pe->d_units;
                        a.nunits = pe->nunits;
                        a.unit_dirs = pe->d_unit_dirs;
                        // one image: units balanced over the SMs (EUCALC_K2_UNIT_BALANCE=0: off)
                        const char *ub = getenv("EUCALC_K2_UNIT_BALANCE");
                        if (cx->batch == 1 && !(ub && ub[0] == '0') &&
                            plan_units_balanced(*pe, num_sms()) == EUCALC_OK && pe->bal_nunits > 0) {
                            a.units = pe->d_bal_units;
                            a.nunits = pe->bal_nunits;
                            a.unit_dirs = pe->d_bal_unit_dirs;
                        }
                        a.stage_base = pe->d_stage_base;
                        a.stage_img = pe->stage_img;
                        a.stage_cap = cx->batch * pe->stage_img;
                        unit = true;
                        // several images: all units of the heaviest image first (EUCALC_K2_IMG_ORDER=0: interleaved)
                        const char *io = getenv("EUCALC_K2_IMG_ORDER");
                        if (cx->batch > 1 && !(io && io[0] == '0')) {
                            std::vector<int64_t> w(cx->batch, 0);
                            for (int64_t b = 0; b < cx->batch; ++b)
                                for (int q = 0; q < cr->Q; ++q) w[b] += cr->h_count[b * cr->Q + q];
                            std::vector<int32_t> ord(cx->batch);
                            std::iota(ord.begin(), ord.end(), 0);
                            std::stable_sort(ord.begin(), ord.end(), [&](int32_t x, int32_t y) { return w[x] > w[y]; });
                            int32_t *d_ord = (int32_t *)dalloc(sizeof(int32_t) * cx->batch);
                            if (d_ord && cudaMemcpyAsync(d_ord, ord.data(), sizeof(int32_t) * cx->batch,
                                                         cudaMemcpyHostToDevice, st) == cudaSuccess)
                                a.img_order = d_ord;  // pageable source: staged before the call returns
                            else
                                cudaGetLastError();
                        }
                    } else {
                        cudaGetLastError();
                    }
                }
            }
        }
        // block regime, one CTA per segment: fixed staging slots per segment (as in the unit
        // path) + k2_scan + k2_unit_copy instead of look-back and copy-out inside the
        // kernel, when the slots (6 arrays x batch x sum of R) fit a memory budget
        // (EUCALC_K2_SLOTS=0: per-CTA staging with look-back)
        bool slots = false;
        {
            const char *ev = getenv("EUCALC_K2_SLOTS");
            if (!unit && !(ev && ev[0] == '0') && k2_block_regime(a) && S >= 2 * (int64_t)num_sms()) {
                s = plan_units(*pe);  // builds the per-direction slot offsets
                if (s != EUCALC_OK) {
                    free_scratch();
                    return s;
                }
                const size_t sb = 6 * (size_t)cx->batch * (size_t)pe->stage_img * esz;
                // budget: 16 GB and an eighth of the device's memory (queried once: cudaMemGetInfo
                // costs ~1 ms per call); a failed allocation falls back to per-CTA staging
                static size_t total_mem[64] = {};
                int dev = 0;
                cudaGetDevice(&dev);
                if (dev >= 0 && dev < 64 && !total_mem[dev]) {
                    size_t free_b = 0, total_b = 0;
                    if (cudaMemGetInfo(&free_b, &total_b) == cudaSuccess) total_mem[dev] = total_b;
                }
                const size_t budget = dev >= 0 && dev < 64 ? total_mem[dev] / 8 : 0;
                if (pe->stage_img > 0 && sb <= (size_t(16) << 30) && sb <= budget) {
                    a.stage = dalloc(sb);
                    if (a.stage) {
                        a.stage_base = pe->d_stage_base;
                        a.stage_img = pe->stage_img;
                        a.stage_cap = cx->batch * pe->stage_img;
                        a.seg_order = pe->d_dir_by_R;
                        slots = true;
                    } else {
                        cudaGetLastError();
                    }
                }
            }
        }
        int64_t scap = 0;
        const size_t sbytes = (unit || slots) ? 0 : k2_stage_bytes(a, num_sms(), &scap);
        if (sbytes) {
            a.stage = dalloc(sbytes);
            a.stage_cap = a.stage ? scap : 0;
            if (!a.stage) cudaGetLastError();  // no staging: the block regime fills twice
        }
        tr.mark("stage");
        ProfScope ps("k2_transforms", st);
        e = launch_k2(a, st, num_sms());
        tr.mark("launch_k2");
        if (e == cudaSuccess && getenv("EUCALC_K2_CHK_BITS")) {  // test hook: read the restart count
            unsigned r = 0;
            e = cudaMemcpyAsync(&r, ticket + 3, sizeof(unsigned), cudaMemcpyDeviceToHost, st);
            if (e == cudaSuccess) e = cudaStreamSynchronize(st);
            g_k2_restarts += r;
        }
    }
    if (e == cudaSuccess && host_out) {
        // copy back: offsets first (to learn the exact totals), then the used entries
        for (int i = 0; i < 3 && e == cudaSuccess; ++i) {
            eucalc_steps *o = outs[i];
            if (!o) continue;
            e = cudaMemcpyAsync(o->offsets, dev[i].off, sizeof(int64_t) * (S + 1), cudaMemcpyDeviceToHost, st);
        }
        if (e == cudaSuccess) e = cudaStreamSynchronize(st);
        for (int i = 0; i < 3 && e == cudaSuccess; ++i) {
            eucalc_steps *o = outs[i];
            if (!o) continue;
            const size_t nbytes = esz * (size_t)o->offsets[S];
            if (nbytes == 0) continue;
            e = cudaMemcpyAsync(o->value, dev[i].v, nbytes, cudaMemcpyDeviceToHost, st);
            if (e == cudaSuccess && o->height && !(i == 2 && cls_alias))
                e = cudaMemcpyAsync(o->height, dev[i].h, nbytes, cudaMemcpyDeviceToHost, st);
        }
    }
    if (e == cudaSuccess && ht_host) e = cudaMemcpyAsync(ht->out, d_ht, ht_osz * S, cudaMemcpyDeviceToHost, st);
    free_scratch();
    arena_trim(st);
    if (e == cudaSuccess && (host_out || ht_host)) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return cuda_fail(e, "transforms");
    return EUCALC_OK;
}

}  // namespace

extern "C" {

eucalc_status eucalc_transforms(const eucalc_critical *cr, const int32_t *dirs, int64_t D, eucalc_steps *ect,
                                eucalc_steps *ordinary, eucalc_steps *classical, int64_t *required_out,
                                void *stream) {
    return transforms_impl(cr, dirs, D, ect, ordinary, classical, nullptr, required_out, stream);
}

eucalc_status eucalc_transforms_ht(const eucalc_critical *cr, const int32_t *dirs, int64_t D, eucalc_steps *ect,
                                   eucalc_steps *ordinary, eucalc_steps *classical, int kernel, double param,
                                   int precision, void *ht_out, int64_t *required_out, void *stream) {
    const HtReq h{kernel, precision, param, ht_out};
    return transforms_impl(cr, dirs, D, ect, ordinary, classical, &h, required_out, stream);
}

eucalc_status eucalc_transforms_real(const eucalc_critical *ccr, const double *dirs, int64_t D, eucalc_steps *ect,
                                     eucalc_steps *ordinary, eucalc_steps *classical, int64_t *required_out,
                                     void *stream) {
    if (!ccr) return fail(EUCALC_E_STATE, "NULL handle");
    eucalc_critical *cr = const_cast<eucalc_critical *>(ccr);
    const Complex *cx = cr->cx;
    const int n = cx->ndim, full = (1 << n) - 1;
    cudaStream_t st = (cudaStream_t)stream;
    cr->users.note(st, cr->owner_stream);
    if (D < 0) return fail(EUCALC_E_ARG, "D < 0");
    if (D > 0 && !dirs) return fail(EUCALC_E_ARG, "dirs is NULL");
    std::vector<double> h((size_t)D * n);
    if (D > 0) {
        if (is_device_ptr(dirs)) {
            CK(cudaMemcpyAsync(h.data(), dirs, sizeof(double) * D * n, cudaMemcpyDeviceToHost, st));
            CK(cudaStreamSynchronize(st));
        } else {
            memcpy(h.data(), dirs, sizeof(double) * D * n);
        }
    }
    std::vector<int32_t> hq(D), hsw(D);
    for (int64_t d = 0; d < D; ++d) {
        int e = 0;
        for (int k = 0; k < n; ++k) {
            const double v = h[d * n + k];
            if (!(v == v) || v == INFINITY || v == -INFINITY) return fail(EUCALC_E_ARG, "direction is not finite");
            if (v == 0.0) {
                g_bad = d;
                return fail(EUCALC_E_NONGENERIC, "direction " + std::to_string(d) + " has a zero coordinate (P:105)");
            }
            if (v > 0) e |= 1 << k;
        }
        const bool rep = ((e >> (n - 1)) & 1) == 0;
        hq[d] = rep ? e : (e ^ full);
        hsw[d] = rep ? 0 : 1;
    }
    eucalc_status s = sync_counts(cr, st);
    if (s != EUCALC_OK) return s;
    // every stream has at most one entry per distinct height <= list length
    int64_t bnd = 0;
    {
        std::vector<int64_t> per_q(cr->Q, 0), dirs_q(cr->Q, 0);
        for (int64_t b = 0; b < cx->batch; ++b)
            for (int q = 0; q < cr->Q; ++q) per_q[q] += cr->h_count[b * cr->Q + q];
        for (int64_t d = 0; d < D; ++d) dirs_q[hq[d]] += 1;
        for (int q = 0; q < cr->Q; ++q) bnd += per_q[q] * dirs_q[q];
    }
    if (required_out) *required_out = bnd;
    eucalc_steps *outs[3] = {ect, ordinary, classical};
    for (eucalc_steps *o : outs) {
        if (!o) continue;
        if (!o->offsets || (!o->height && o != classical) || !o->value) return fail(EUCALC_E_ARG, "NULL output array");
        if (o->elem_bytes != 8) return fail(EUCALC_E_ARG, "real-valued directions need elem_bytes 8 (double heights, int64 values)");
        if (o->capacity < bnd) return fail(EUCALC_E_CAPACITY, "capacity " + std::to_string(o->capacity) + " < required bound " + std::to_string(bnd));
    }
    if (!ect && !ordinary && !classical) return EUCALC_OK;
    if (cr->max_abs_sum >= (int64_t(1) << 31)) return fail(EUCALC_E_RANGE, "total |weight| of a critical list exceeds 2^31");
    const int64_t S = cx->batch * D;
    if (S == 0) return EUCALC_OK;
    // the warp-regime loops step int32 segment indices by the grid's warp count
    // (< 2^24): keep s + step below 2^31
    if (S > INT32_MAX - (int64_t(1) << 24))
        return fail(EUCALC_E_RANGE, "more than 2^31 - 2^24 (image, direction) segments in one call");
    const bool cls_alias = classical && ect && (classical->height == ect->height || !classical->height);
    if (classical && !classical->height && !ect) return fail(EUCALC_E_ARG, "classical height is NULL");
    bool host_out = false;
    for (eucalc_steps *o : outs)
        if (o && !is_device_ptr(o->value)) host_out = true;
    std::vector<void *> scratch;
    auto dalloc = [&](size_t bytes) -> void * {
        void *q = nullptr;
        if (cudaMallocAsync(&q, std::max<size_t>(bytes, 1), st) != cudaSuccess) return nullptr;
        scratch.push_back(q);
        return q;
    };
    auto free_scratch = [&]() { for (void *q : scratch) cudaFreeAsync(q, st); };
    StepsOut dev[3] = {};
    for (int i = 0; i < 3; ++i) {
        eucalc_steps *o = outs[i];
        if (!o) continue;
        if (host_out) {
            dev[i].off = (int64_t *)dalloc(sizeof(int64_t) * (S + 1));
            dev[i].v = dalloc(8 * (size_t)std::max<int64_t>(bnd, 1));
            dev[i].h = (i == 2 && cls_alias) ? dev[0].h : dalloc(8 * (size_t)std::max<int64_t>(bnd, 1));
            if (!dev[i].off || !dev[i].v || !dev[i].h) {
                free_scratch();
                return fail(EUCALC_E_NOMEM, "device scratch for host outputs");
            }
        } else {
            dev[i].off = o->offsets;
            dev[i].h = (i == 2 && cls_alias) ? nullptr : o->height;
            dev[i].v = o->value;
        }
    }
    // Lists longer than kSmallMax take the bucketed path (K5Big): planned here in
    // segment order and cut into chunks whose scratch fits a memory budget.
    // (EUCALC_K5_SMALL_MAX / EUCALC_K5_BUCKET: test hooks that force the bucketed
    // path, and oversize pieces, on inputs small enough for the oracle)
    int64_t kSmallMax = 4096, bucket = kK5Bucket;
    if (const char *v = getenv("EUCALC_K5_SMALL_MAX")) kSmallMax = std::min<int64_t>(4096, std::max<int64_t>(0, atoll(v)));
    if (const char *v = getenv("EUCALC_K5_BUCKET")) bucket = std::max<int64_t>(1, atoll(v));
    int64_t small_np = 0;
    std::vector<int64_t> g_seg, g_pbase, g_sbase;
    std::vector<int32_t> g_nb;
    struct Chunk {
        int64_t i0, i1, npieces, nrec;
        int nb_max;
    };
    std::vector<Chunk> chunks;
    {
        size_t fr = 0, tot = 0;
        if (cudaMemGetInfo(&fr, &tot) != cudaSuccess) fr = size_t(4) << 30;
        const int64_t budget_rec = std::max<int64_t>(1, (int64_t)(std::min<size_t>(fr / 4, size_t(8) << 30) / 32));
        Chunk cur{0, 0, 0, 0, 0};
        for (int64_t b = 0; b < cx->batch; ++b)
            for (int64_t d = 0; d < D; ++d) {
                const int64_t nrec = cr->h_count[b * cr->Q + hq[d]];
                if (nrec <= kSmallMax) {
                    small_np = std::max(small_np, nrec);
                    continue;
                }
                const int32_t nb = (int32_t)std::min<int64_t>(kK5MaxBuckets, (nrec + bucket - 1) / bucket);
                if (cur.i1 > cur.i0 && cur.nrec + nrec > budget_rec) {
                    chunks.push_back(cur);
                    cur = Chunk{cur.i1, cur.i1, 0, 0, 0};
                }
                g_seg.push_back(b * D + d);
                g_pbase.push_back(cur.npieces);
                g_sbase.push_back(cur.nrec);
                g_nb.push_back(nb);
                cur.i1 += 1;
                cur.npieces += nb;
                cur.nrec += nrec;
                cur.nb_max = std::max(cur.nb_max, (int)nb);
            }
        if (cur.i1 > cur.i0) chunks.push_back(cur);
    }
    const int64_t nbig = (int64_t)g_seg.size();
    int64_t max_rec = 0, max_p = 0;
    for (const Chunk &c : chunks) {
        max_rec = std::max(max_rec, c.nrec);
        max_p = std::max(max_p, c.npieces);
    }
    double *d_xi = (double *)dalloc(sizeof(double) * D * n);
    int32_t *d_q = (int32_t *)dalloc(sizeof(int32_t) * D), *d_sw = (int32_t *)dalloc(sizeof(int32_t) * D);
    unsigned long long *flags = (unsigned long long *)dalloc(sizeof(unsigned long long) * S);
    unsigned int *ticket = (unsigned int *)dalloc(sizeof(unsigned int) * 4);
    int *cnts = (int *)dalloc(sizeof(int) * 2 * S);
    if (!d_xi || !d_q || !d_sw || !flags || !ticket || !cnts) {
        free_scratch();
        return fail(EUCALC_E_NOMEM, "scratch");
    }
    K5Big big{};
    int64_t *d_gseg = nullptr, *d_gpbase = nullptr, *d_gsbase = nullptr;
    int32_t *d_gnb = nullptr;
    if (nbig > 0) {
        d_gseg = (int64_t *)dalloc(sizeof(int64_t) * nbig);
        d_gpbase = (int64_t *)dalloc(sizeof(int64_t) * nbig);
        d_gsbase = (int64_t *)dalloc(sizeof(int64_t) * nbig);
        d_gnb = (int32_t *)dalloc(sizeof(int32_t) * nbig);
        big.scr = (uint4 *)dalloc(16 * (size_t)max_rec);
        big.tmp = (uint4 *)dalloc(16 * (size_t)max_rec);
        big.p_start = (int64_t *)dalloc(sizeof(int64_t) * max_p);
        int32_t *pa = (int32_t *)dalloc(sizeof(int32_t) * max_p * 11);
        big.over = (unsigned *)dalloc(sizeof(unsigned) * (2 + max_p));
        if (!d_gseg || !d_gpbase || !d_gsbase || !d_gnb || !big.scr || !big.tmp || !big.p_start || !pa || !big.over) {
            free_scratch();
            return fail(EUCALC_E_NOMEM, "scratch for long lists");
        }
        int32_t **arr[11] = {&big.p_len, &big.p_seg, &big.p_nc, &big.p_no, &big.p_sc, &big.p_sj,
                             &big.p_offc, &big.p_offo, &big.p_ic, &big.p_ij, nullptr};
        for (int k = 0; k < 10; ++k) *arr[k] = pa + (size_t)k * max_p;
        big.over_cap = max_p;
    }
    cudaError_t e = cudaMemcpyAsync(d_xi, h.data(), sizeof(double) * D * n, cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(d_q, hq.data(), sizeof(int32_t) * D, cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(d_sw, hsw.data(), sizeof(int32_t) * D, cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess && nbig > 0) {
        e = cudaMemcpyAsync(d_gseg, g_seg.data(), sizeof(int64_t) * nbig, cudaMemcpyHostToDevice, st);
        if (e == cudaSuccess) e = cudaMemcpyAsync(d_gpbase, g_pbase.data(), sizeof(int64_t) * nbig, cudaMemcpyHostToDevice, st);
        if (e == cudaSuccess) e = cudaMemcpyAsync(d_gsbase, g_sbase.data(), sizeof(int64_t) * nbig, cudaMemcpyHostToDevice, st);
        if (e == cudaSuccess) e = cudaMemcpyAsync(d_gnb, g_nb.data(), sizeof(int32_t) * nbig, cudaMemcpyHostToDevice, st);
    }
    if (e == cudaSuccess) e = cudaMemsetAsync(flags, 0, sizeof(unsigned long long) * S, st);
    if (e == cudaSuccess) e = cudaMemsetAsync(ticket, 0, sizeof(unsigned int) * 4, st);
    if (e == cudaSuccess) {
        K5Args a{};
        a.rec = cr->d_rec;
        a.wide = cr->wide;
        a.vcap = cr->vcap;
        a.count = cr->d_count;
        a.Q = cr->Q;
        a.ndim = n;
        for (int k = 0; k < n; ++k) {
            a.sh[k] = cx->sh[k];
            a.msk[k] = cx->msk[k];
            a.M[k] = (int)cx->M[k];
        }
        a.xi = d_xi;
        a.q = d_q;
        a.swap = d_sw;
        a.D = D;
        a.batch = cx->batch;
        int np2 = 32;
        while (np2 < small_np) np2 <<= 1;
        a.npow2 = np2;
        a.small_max = (int)kSmallMax;
        a.cnt_c = cnts;
        a.cnt_o = cnts + S;
        a.do_ect = ect != nullptr;
        a.do_ord = ordinary != nullptr;
        a.do_cls = classical != nullptr;
        a.cls_alias = cls_alias;
        a.ect = dev[0];
        a.ord = dev[1];
        a.cls = dev[2];
        a.scan.do_ect = a.do_ect;
        a.scan.do_ord = a.do_ord;
        a.scan.do_cls = a.do_cls;
        a.scan.ect = dev[0];
        a.scan.ord = dev[1];
        a.scan.cls = dev[2];
        a.scan.flags = flags;
        a.scan.ticket = ticket;
        ProfScope ps("k5_real", st);
        const int sms = num_sms();
        auto chunk_big = [&](const Chunk &c) {
            K5Big g = big;
            g.seg = d_gseg + c.i0;
            g.pbase = d_gpbase + c.i0;
            g.sbase = d_gsbase + c.i0;
            g.nb = d_gnb + c.i0;
            g.nseg = c.i1 - c.i0;
            g.npieces = c.npieces;
            return g;
        };
        // one chunk: its sorted pieces stay in scratch for the emit pass; several
        // chunks: counts in a first round, everything redone per chunk to emit
        for (size_t c = 0; c < chunks.size() && e == cudaSuccess; ++c)
            e = launch_k5b_prepare(a, chunk_big(chunks[c]), chunks[c].nb_max, st, sms);
        if (e == cudaSuccess) e = launch_k5(a, 0, st, sms);
        if (e == cudaSuccess) e = launch_k5_scan(a, st);
        if (e == cudaSuccess) e = launch_k5(a, 1, st, sms);
        for (size_t c = 0; c < chunks.size() && e == cudaSuccess; ++c) {
            if (chunks.size() > 1) e = launch_k5b_prepare(a, chunk_big(chunks[c]), chunks[c].nb_max, st, sms);
            if (e == cudaSuccess) e = launch_k5b_emit(a, chunk_big(chunks[c]), st, sms);
        }
    }
    if (e == cudaSuccess && host_out) {
        for (int i = 0; i < 3 && e == cudaSuccess; ++i) {
            eucalc_steps *o = outs[i];
            if (!o) continue;
            e = cudaMemcpyAsync(o->offsets, dev[i].off, sizeof(int64_t) * (S + 1), cudaMemcpyDeviceToHost, st);
        }
        if (e == cudaSuccess) e = cudaStreamSynchronize(st);
        for (int i = 0; i < 3 && e == cudaSuccess; ++i) {
            eucalc_steps *o = outs[i];
            if (!o) continue;
            const size_t nbytes = 8 * (size_t)o->offsets[S];
            if (nbytes == 0) continue;
            e = cudaMemcpyAsync(o->value, dev[i].v, nbytes, cudaMemcpyDeviceToHost, st);
            if (e == cudaSuccess && o->height && !(i == 2 && cls_alias))
                e = cudaMemcpyAsync(o->height, dev[i].h, nbytes, cudaMemcpyDeviceToHost, st);
        }
    }
    free_scratch();
    if (e == cudaSuccess && host_out) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return cuda_fail(e, "transforms_real");
    return EUCALC_OK;
}

eucalc_status eucalc_ect(const eucalc_critical *cr, const int32_t *dirs, int64_t D, eucalc_steps *ect,
                         int64_t *required_out, void *stream) {
    if (!ect) return fail(EUCALC_E_ARG, "ect is NULL");
    return eucalc_transforms(cr, dirs, D, ect, nullptr, nullptr, required_out, stream);
}

eucalc_status eucalc_radon(const eucalc_critical *cr, const int32_t *dirs, int64_t D, eucalc_steps *ordinary,
                           eucalc_steps *classical, int64_t *required_out, void *stream) {
    if (!ordinary || !classical) return fail(EUCALC_E_ARG, "ordinary/classical is NULL");
    if (!classical->height) return fail(EUCALC_E_ARG, "classical height is NULL");
    return eucalc_transforms(cr, dirs, D, nullptr, ordinary, classical, required_out, stream);
}

eucalc_status eucalc_hybrid(const eucalc_critical *ccr, const int32_t *dirs, int64_t D, int kernel, double param,
                            int precision, void *out, void *stream) {
    return eucalc_hybrid_ex(ccr, dirs, D, kernel, param, precision, EUCALC_HT_AUTO, out, stream);
}

eucalc_status eucalc_hybrid_ex(const eucalc_critical *ccr, const int32_t *dirs, int64_t D, int kernel, double param,
                               int precision, int algorithm, void *out, void *stream) {
    if (!ccr) return fail(EUCALC_E_STATE, "NULL handle");
    if (algorithm < EUCALC_HT_AUTO || algorithm > EUCALC_HT_TABLE) return fail(EUCALC_E_ARG, "bad algorithm");
    if (kernel < EUCALC_K_GAUSS || kernel > EUCALC_K_EXP) return fail(EUCALC_E_ARG, "bad kernel");
    if (precision != EUCALC_F32 && precision != EUCALC_F64) return fail(EUCALC_E_ARG, "bad precision");
    if ((kernel == EUCALC_K_GAUSS || kernel == EUCALC_K_COS) && !(param > 0)) return fail(EUCALC_E_ARG, "param must be > 0");
    if (D > 0 && !out) return fail(EUCALC_E_ARG, "out is NULL");
    eucalc_critical *cr = const_cast<eucalc_critical *>(ccr);
    const Complex *cx = cr->cx;
    cudaStream_t st = (cudaStream_t)stream;
    cr->users.note(st, cr->owner_stream);
    std::shared_ptr<PlanEntry> pe;
    eucalc_status s = get_plan(cx, dirs, D, st, pe);
    if (s != EUCALC_OK) return s;
    const DirPlan &p = pe->p;
    s = sync_counts(cr, st);
    if (s != EUCALC_OK) return s;
    if (D == 0) return EUCALC_OK;
    const std::vector<int32_t> &tstart = pe->tstart;
    // tabulated kbar when the packed-coordinate height (dp2a/dp4a) applies and the
    // half table of one u-parity fits shared memory; else per-term evaluation
    const int64_t U = p.U1 - p.U0 + 1;
    const bool table_ok = p.dp != 0 && U < (int64_t(1) << 30) &&
                          k3_table_smem(k3_mode(kernel, precision, cr->wide), U) <= 200 * 1024;
    if (algorithm == EUCALC_HT_TABLE && !table_ok)
        return fail(EUCALC_E_ARG, "tabulated HT needs byte-aligned coordinates, |xs| <= 127 and a table that fits shared memory");
    const bool use_table = algorithm == EUCALC_HT_TABLE || (algorithm == EUCALC_HT_AUTO && table_ok);
    // records per CTA: the kernel's chunk, shrunk (to >= 512) when the grid would
    // not cover the SMs twice (few images / tiles, e.g. one large image)
    int chunk = k3_chunk(use_table);
    const int64_t ctas_per_chunk = (int64_t)pe->tstart.size() * cx->batch;
    while (chunk > 512 && ctas_per_chunk * ((cr->max_count + chunk - 1) / chunk) < 2 * num_sms()) chunk /= 2;
    const int nchunks = (int)std::max<int64_t>(1, (cr->max_count + chunk - 1) / chunk);
    const size_t osz = precision == EUCALC_F32 ? 4 : 8;
    const bool host_out = !is_device_ptr(out);
    std::vector<void *> scratch;
    
    auto free_scratch = [&]() { for (void *q : scratch) cudaFreeAsync(q, st); };
    const DirInfo *d_info = pe->d_info;
    const int32_t *d_order = pe->d_order, *d_ts = pe->d_ts, *d_tl = pe->d_tl, *d_cs = pe->d_csum;
    std::vector<void *> ar;
    if (!arena_take(st, {sizeof(double) * cx->batch * nchunks * D, host_out ? osz * cx->batch * D : 0,
                         use_table ? 12 * (size_t)U : 0},
                    ar)) {
        free_scratch();
        return fail(EUCALC_E_NOMEM, "scratch");
    }
    double *d_part = (double *)ar[0];
    void *d_out = host_out ? ar[1] : out;
    void *d_tab = ar[2];
    if (!d_part || !d_out || (use_table && !d_tab)) {
        free_scratch();
        return fail(EUCALC_E_NOMEM, "scratch");
    }
    cudaError_t e = cudaSuccess;
    if (e == cudaSuccess) {
        K3Args a{};
        a.rec = cr->d_rec;
        a.wide = cr->wide;
        a.vcap = cr->vcap;
        a.count = cr->d_count;
        a.Q = cr->Q;
        a.ndim = cx->ndim;
        for (int k = 0; k < cx->ndim; ++k) {
            a.sh[k] = cx->sh[k];
            a.msk[k] = cx->msk[k];
        }
        a.dirs = d_info;
        a.order = d_order;
        a.tile_start = d_ts;
        a.tile_len = d_tl;
        a.ntiles = (int)tstart.size();
        a.D = D;
        a.batch = cx->batch;
        a.kernel = kernel;
        a.precision = precision;
        a.param = param;
        a.L = cx->L;
        a.csum = d_cs;
        a.dp = p.dp;
        const int maxlen = *std::max_element(pe->tlen.begin(), pe->tlen.end());
        a.threads = std::max(32, (maxlen + 31) / 32 * 32);
        a.nchunks = nchunks;
        a.chunk = chunk;
        a.partial = d_part;
        a.out = d_out;
        a.use_table = use_table ? 1 : 0;
        a.U0 = p.U0;
        a.U = U;
        a.tab64 = (double *)d_tab;
        a.tab32 = use_table ? (float *)((double *)d_tab + U) : nullptr;
        ProfScope ps("k3_hybrid", st);
        e = launch_k3(a, st);
    }
    if (e == cudaSuccess && host_out) e = cudaMemcpyAsync(out, d_out, osz * cx->batch * D, cudaMemcpyDeviceToHost, st);
    free_scratch();
    arena_trim(st);
    if (e == cudaSuccess && host_out) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return cuda_fail(e, "hybrid");
    return EUCALC_OK;
}

}  // extern "C"

namespace {

// Shared body of eucalc_evaluate / eucalc_vectorize (K4).
eucalc_status eval_common(const eucalc_complex *cx, const int32_t *dirs, int64_t D, int kind, const eucalc_steps *rep,
                          const eucalc_steps *cls, const double *t, double ta, double tb, int64_t nq, void *out,
                          int out_eb, void *stream) {
    if (!cx || !cx->d_img) return fail(EUCALC_E_STATE, "invalid complex");
    if (kind != EUCALC_EVAL_ECT && kind != EUCALC_EVAL_RADON) return fail(EUCALC_E_ARG, "bad kind");
    if (!rep || !rep->offsets || !rep->height || !rep->value) return fail(EUCALC_E_ARG, "NULL representation");
    if (kind == EUCALC_EVAL_RADON && (!cls || !cls->offsets || !cls->height || !cls->value))
        return fail(EUCALC_E_ARG, "Radon evaluation needs the classical stream");
    const int in_eb = rep->elem_bytes;
    if (in_eb != 2 && in_eb != 4 && in_eb != 8) return fail(EUCALC_E_ARG, "elem_bytes must be 2, 4 or 8");
    if (kind == EUCALC_EVAL_RADON && cls->elem_bytes != in_eb) return fail(EUCALC_E_ARG, "rep/classical elem_bytes differ");
    if (out_eb != 4 && out_eb != 8) return fail(EUCALC_E_ARG, "out_elem_bytes must be 4 or 8");
    if (out_eb == 4 && in_eb == 8) return fail(EUCALC_E_ARG, "int32 output of an int64 representation");
    if (nq < 0) return fail(EUCALC_E_ARG, "negative query count");
    if (nq > 0 && !out) return fail(EUCALC_E_ARG, "out is NULL");
    if (t == nullptr && (ta != ta || tb != tb)) return fail(EUCALC_E_ARG, "NaN interval bound");
    cudaStream_t st = (cudaStream_t)stream;
    std::shared_ptr<PlanEntry> pe;
    eucalc_status s = get_plan(cx, dirs, D, st, pe);
    if (s != EUCALC_OK) return s;
    const int64_t S = cx->batch * D;
    if (S == 0 || nq == 0) return EUCALC_OK;
    std::vector<void *> scratch;
    auto dalloc = [&](size_t bytes) -> void * {
        void *q = nullptr;
        if (cudaMallocAsync(&q, std::max<size_t>(bytes, 1), st) != cudaSuccess) return nullptr;
        scratch.push_back(q);
        return q;
    };
    auto free_scratch = [&]() { for (void *q : scratch) cudaFreeAsync(q, st); };
    // representations: device pointers used in place; host CSR staged to the device
    struct Dev { const int64_t *off; const void *h, *v; };
    auto stage = [&](const eucalc_steps *r, Dev &d) -> eucalc_status {
        if (is_device_ptr(r->offsets)) {
            d = Dev{r->offsets, r->height, r->value};
            return EUCALC_OK;
        }
        const int64_t n = r->offsets[S] - r->offsets[0];
        if (n < 0 || r->offsets[0] != 0) return fail(EUCALC_E_ARG, "bad host offsets");
        void *o = dalloc(sizeof(int64_t) * (S + 1)), *h = dalloc(in_eb * n), *v = dalloc(in_eb * n);
        if (!o || !h || !v) return fail(EUCALC_E_NOMEM, "evaluation staging");
        cudaError_t e = cudaMemcpyAsync(o, r->offsets, sizeof(int64_t) * (S + 1), cudaMemcpyHostToDevice, st);
        if (e == cudaSuccess && n) e = cudaMemcpyAsync(h, r->height, in_eb * n, cudaMemcpyHostToDevice, st);
        if (e == cudaSuccess && n) e = cudaMemcpyAsync(v, r->value, in_eb * n, cudaMemcpyHostToDevice, st);
        if (e != cudaSuccess) return cuda_fail(e, "evaluation staging");
        d = Dev{(const int64_t *)o, h, v};
        return EUCALC_OK;
    };
    Dev dr{}, dc{};
    s = stage(rep, dr);
    if (s == EUCALC_OK && kind == EUCALC_EVAL_RADON) s = stage(cls, dc);
    const double *d_t = t;
    if (s == EUCALC_OK && t && !is_device_ptr(t)) {
        double *q = (double *)dalloc(sizeof(double) * nq);
        if (!q) s = fail(EUCALC_E_NOMEM, "query staging");
        else if (cudaMemcpyAsync(q, t, sizeof(double) * nq, cudaMemcpyHostToDevice, st) != cudaSuccess)
            s = fail(EUCALC_E_CUDA, "query staging");
        d_t = q;
    }
    const bool host_out = !is_device_ptr(out);
    void *d_out = out;
    if (s == EUCALC_OK && host_out) {
        d_out = dalloc((size_t)out_eb * S * nq);
        if (!d_out) s = fail(EUCALC_E_NOMEM, "output staging");
    }
    if (s != EUCALC_OK) {
        free_scratch();
        cudaStreamSynchronize(st);
        return s;
    }
    K4Args a{};
    a.kind = kind;
    a.rep_off = dr.off;
    a.rep_h = dr.h;
    a.rep_v = dr.v;
    a.cls_off = dc.off;
    a.cls_h = dc.h;
    a.cls_v = dc.v;
    a.in_eb = in_eb;
    a.out_eb = out_eb;
    a.L = cx->L;
    a.csum = pe->d_csum;
    a.D = D;
    a.batch = cx->batch;
    a.t = d_t;
    a.ta = ta;
    a.tb = tb;
    a.nq = nq;
    a.out = d_out;
    cudaError_t e;
    {
        ProfScope ps("k4_evaluate", st);
        e = launch_k4(a, st, num_sms());
    }
    if (e == cudaSuccess && host_out) e = cudaMemcpyAsync(out, d_out, (size_t)out_eb * S * nq, cudaMemcpyDeviceToHost, st);
    free_scratch();
    if (e == cudaSuccess && host_out) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return cuda_fail(e, "evaluate");
    return EUCALC_OK;
}

}  // namespace

extern "C" {

eucalc_status eucalc_evaluate(const eucalc_complex *cx, const int32_t *dirs, int64_t D, int kind,
                              const eucalc_steps *rep, const eucalc_steps *classical, const double *t, int64_t nq,
                              void *out, int out_elem_bytes, void *stream) {
    if (nq > 0 && !t) return fail(EUCALC_E_ARG, "t is NULL");
    return eval_common(cx, dirs, D, kind, rep, classical, t, 0.0, 0.0, nq, out, out_elem_bytes, stream);
}

eucalc_status eucalc_vectorize(const eucalc_complex *cx, const int32_t *dirs, int64_t D, int kind,
                               const eucalc_steps *rep, const eucalc_steps *classical, double a, double b, int64_t N,
                               void *out, int out_elem_bytes, void *stream) {
    if (N < 0) return fail(EUCALC_E_ARG, "N < 0");
    return eval_common(cx, dirs, D, kind, rep, classical, nullptr, a, b, N, out, out_elem_bytes, stream);
}

eucalc_status eucalc_height_map(const eucalc_complex *cx, const int32_t *dir, int64_t *L, int64_t *csum) {
    if (!cx || !dir) return fail(EUCALC_E_ARG, "NULL argument");
    int64_t cs = 0;
    for (int k = 0; k < cx->ndim; ++k)
        if (cx->M[k] > 1) cs += dir[k];
    if (L) *L = cx->L;
    if (csum) *csum = cs;
    return EUCALC_OK;
}

}  // extern "C"
