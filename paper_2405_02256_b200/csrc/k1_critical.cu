// K1 — critical points (SURVEY 8(a) A1 stencil + A2 ordered compaction).
//
// For every vertex x of every image and every sign vector eps:
//   Delta^-(eps, x) = chi(phi | lwst(eps, x))
// where the lower star is the set of cells at doubled coordinates 2x - delta o eps,
// delta in {0,1}^n, restricted to existing cells (E16):
//   VERTEX: phi(cell) = min of its vertices; the cell exists iff all of
//                   its vertices do (out-of-range vertex = lowest sentinel);
//   TOP: phi(cell) = min over its top cofaces (pixels); out-of-range
//                   pixel = highest sentinel, so a cell whose fixed pixel index is
//                   out of range does not exist while a border face keeps the min
//                   of its real cofaces.
// Per vertex the 3^n star values are box mins of the neighbourhood, masked to 0
// where the cell does not exist, and the 2^n lower-star sums come from an
// inclusion-exclusion transform along every axis.
//
// Compaction: per antipodal pair {eps, -eps} (eps the representative with
// eps_{n-1} = -1) a vertex is kept iff Delta^-(eps) != 0 or Delta^-(-eps) != 0
// (this covers the classical points of both orthants and every ordinary point,
// since J(eps) = Delta^-(eps) - Delta^-(-eps)).
//
// Work decomposition ("pencils"): one warp owns 32 consecutive vertices of the
// fastest axis x (one per lane) and walks the slowest axis (z in 3-D, y in 2-D)
// plane by plane, so the stencil is separable along the walk: each step loads
// only the new plane's neighbourhood (each lane its own column, x +- 1 by warp
// shuffles), and for VERTEX the box mins and the inclusion-exclusion of the two
// planes it already saw are carried in registers. There is no shared memory and
// no block barrier on the hot path.
//
// Deterministic order without a look-back or a second stencil pass:
//   k1_pencil<EMIT>: each (tile, warp) writes its kept vertices, in walk order and
//                    lane order (ballot prefix), into its own fixed-capacity region
//                    of scratch lists (capacity = its vertex count, so no overflow),
//                    and its count per pair (+ sum and max of |Delta^-| over the
//                    list, for the host's width choices);
//   k1_scan         : per (image, pair) list, exclusive scan of the region counts in
//                    (tile, warp) order -> each region's list offset, the per-tile
//                    offsets K2 uses to cull tiles, and the list length;
//   k1_copy         : every region's records to their offset (a memory copy).
// Images that are a single region (2-D images of <= 32 x 64 vertices) are
// written in place by k1_pencil alone.
// Tiles (K2's culling unit) are boxes of 32 x 8 x 8 vertices in 3-D (8 warps =
// 8 rows, each walking 8 planes) and 32 x 64 in 2-D (one warp walking 64 rows);
// a list is ordered by tile (x fastest, then y, then z), then warp (row), then
// walk step, then lane. The per-orthant counts N^-, N^ord are a third,
// on-demand variant (k1_pencil<STATS>, eucalc_critical_counts).
#include <algorithm>
#include <climits>
#include <type_traits>

#include "eucalc_internal.cuh"

namespace eucalc {
namespace {

constexpr int kWarps = 8, kThreads = 32 * kWarps;
constexpr int kWalk3 = 64;  // planes walked by one warp in 3-D (8 tiles deep)
// tile geometry (k1_geometry): 3-D 32 x 8 x 8 (8 warps = rows, 8 planes); 2-D 32 x 64,
// walked by a.W warps of 64 / a.W rows each (W = 1 when the image is one tile: then
// it is one region and its lists are written in place; else W = 4, so a 2-D image
// offers 4 pencils per tile)
template <int N> struct Tile;
template <> struct Tile<3> { static constexpr int TY = 8, TZ = 8, W = 8, SEG = 8; };
template <> struct Tile<2> { static constexpr int TY = 64, TZ = 1; };
constexpr int kEmit = 0, kStats = 1;

__host__ __device__ constexpr int pow3(int k) { return k == 0 ? 1 : 3 * pow3(k - 1); }

// Compile-time loop: f(std::integral_constant<int, I>) for I in [B, E). Every
// index below is a constant expression, so the star values stay in registers.
template <int B, int E, typename F>
__device__ __forceinline__ void static_for(F &&f) {
    if constexpr (B < E) {
        f(std::integral_constant<int, B>{});
        static_for<B + 1, E>(f);
    }
}

// digit k (axis k, 0 = slowest) of a base-3 star index, in {0,1,2} <-> offset {-1,0,+1}
template <int N>
__host__ __device__ constexpr int digit3(int idx, int k) { return (idx / pow3(N - 1 - k)) % 3; }

// Does pixel corner c (bit k set <-> pixel index x_k, clear <-> x_k - 1) belong to
// the top-cell cofaces of the star cell `idx` (TOP construction)?
template <int N>
__host__ __device__ constexpr bool top_coface(int idx, int c) {
    for (int k = 0; k < N; ++k) {
        const int o = digit3<N>(idx, k) - 1, cb = (c >> k) & 1;
        if (o == -1 && cb != 0) return false;  // cell extends to x-1: pixel x-1 only
        if (o == 1 && cb != 1) return false;   // cell extends to x+1: pixel x only
    }
    return true;
}

// Inclusion-exclusion along every axis of a 3^M array of masked cell values:
// slot +1 <- v(0) - v(-1) (eps_k = +1), slot -1 <- v(0) - v(+1) (eps_k = -1).
// Corner (digits 0/2 per axis) then holds the lower-star sum of that sign vector.
template <int M>
__device__ __forceinline__ void incl_excl(int (&v)[pow3(M)]) {
    static_for<0, M>([&](auto K) {
        constexpr int k = decltype(K)::value, st = pow3(M - 1 - k);
        static_for<0, pow3(M)>([&](auto I) {
            constexpr int idx = decltype(I)::value;
            if constexpr (digit3<M>(idx, k) == 1) {
                const int a = v[idx - st], c = v[idx], b = v[idx + st];
                v[idx + st] = c - a;
                v[idx - st] = c - b;
            }
        });
    });
}

// corner of a 3^M array for in-plane sign bits `bits` (bit j <-> in-plane axis j,
// j = 0 the slowest): digit 2 where the bit is set, 0 where clear
template <int M>
__host__ __device__ constexpr int corner(int bits) {
    int idx = 0;
    for (int j = 0; j < M; ++j) idx += (((bits >> j) & 1) ? 2 : 0) * pow3(M - 1 - j);
    return idx;
}

// Element type of the sentinel-carrying values: int16 suffices for 8-bit images.
template <int CONS, typename TIn>
struct Sent {
    // VERTEX: lowest (a missing vertex makes the cell's min the sentinel);
    // TOP: highest (a missing pixel drops out of the min)
    static constexpr int value = CONS == EUCALC_VERTEX ? (sizeof(TIn) == 1 ? -1 : INT_MIN) : INT_MAX;
};

// Masked cell value: VERTEX 8-bit images hold values >= 0 > sentinel -1, so one
// max masks (and commutes with min, so it can be applied before the walk's min);
// otherwise compare with the sentinel.
template <int CONS, typename TIn>
__device__ __forceinline__ int mask_cell(int v) {
    if constexpr (CONS == EUCALC_VERTEX && sizeof(TIn) == 1) return max(v, 0);
    else return v == Sent<CONS, TIn>::value ? 0 : v;
}

struct Geo {
    int MX, MY, MZ;  // vertex extents of the (x, y, z) view (MY = 1 in 1-D, MZ = 1 in 2-D)
    int mX, mY, mZ;  // pixel extents
};

// One row of the current plane: each lane's value at x and its neighbours x - 1
// and x + 1 (warp shuffles; lanes 0 / 31 load the halo). Values outside the image
// are the sentinel. `row_ok` is warp-uniform.
template <typename TIn, bool RIGHT>
__device__ __forceinline__ void load_row(const TIn *row, bool row_ok, int x, int ext, int sent, int &l, int &m,
                                         int &r) {
    const int lane = threadIdx.x & 31;
    const int hx = lane == 0 ? x - 1 : x + 1;
    const bool hlane = lane == 0 || (RIGHT && lane == 31);
    int v = sent, hv = sent;
    if (row_ok && x < ext) v = (int)__ldg(row + x);
    if (row_ok && hlane && (unsigned)hx < (unsigned)ext) hv = (int)__ldg(row + hx);
    m = v;
    l = __shfl_up_sync(0xffffffffu, v, 1);
    l = lane == 0 ? hv : l;
    if constexpr (RIGHT) {
        r = __shfl_down_sync(0xffffffffu, v, 1);
        r = lane == 31 ? hv : r;
    }
}

// ------------------------------------------------------------------ VERTEX walk
// Walk state of one lane (vertex column x, row y): the in-plane box mins of the
// current plane w (pm, 3^(N-1) values, unmasked unless the mask commutes), the
// inclusion-exclusion corners of the cells spanning planes w-1 .. w (tlow) and
// the raw values of plane w+1, loaded one step ahead (the walk is latency-bound
// otherwise: the load is then in flight for a whole step).
template <int N>
struct Raw {
    static constexpr int R = N == 3 ? 3 : 1;  // in-plane rows: y-1, y, y+1 (3-D) / the row (2-D)
    int m[R];  // this lane's column
    int h[R];  // halo column: lane 0 holds x - 1, lane 31 holds x + 1
};


// Loads of consecutive planes for one lane: a pointer at (plane p, row y-1, column
// x) advanced one plane per load; row / column validity fixed per lane. Sentinel
// outside the image (predicated loads, nothing dereferenced out of range).
template <int N, typename TIn>
struct PlaneCursor;
template <int N, typename TIn>
struct PlaneCursor {
    const TIn *ptr;
    long long pstride;  // elements per plane
    int rstride;        // elements per row (3-D)
    int p, pend;        // next plane, plane extent
    int hdx;            // halo column offset: -1 (lane 0), +1 (lane 31)
    bool rok[N == 3 ? 3 : 1], xok, hok;
    __device__ __forceinline__ void init(const TIn *img, const Geo &g, int p0, int y, int x) {
        const int lane = threadIdx.x & 31;
        hdx = lane == 0 ? -1 : 1;
        xok = x < g.MX;
        hok = (lane == 0 || lane == 31) && (unsigned)(x + hdx) < (unsigned)g.MX;
        p = p0;
        if constexpr (N == 3) {
            pend = g.MZ;
            pstride = (long long)g.MY * g.MX;
            rstride = g.MX;
            for (int k = 0; k < 3; ++k) rok[k] = (unsigned)(y - 1 + k) < (unsigned)g.MY;
            ptr = img + (long long)p0 * pstride + (long long)(y - 1) * g.MX + x;
        } else {
            pend = g.MY;
            pstride = g.MX;
            rstride = 0;
            rok[0] = true;
            ptr = img + (long long)p0 * g.MX + x;
        }
    }
    __device__ __forceinline__ void load(int sent, Raw<N> &r) {
        const bool pok = (unsigned)p < (unsigned)pend;
#pragma unroll
        for (int k = 0; k < Raw<N>::R; ++k) {
            const TIn *row = ptr + k * rstride;
            int v = sent, hv = sent;
            if (pok && rok[k] && xok) v = (int)__ldg(row);
            if (pok && rok[k] && hok) hv = (int)__ldg(row + hdx);
            r.m[k] = v;
            r.h[k] = hv;
        }
        ptr += pstride;
        ++p;
    }
};

template <int N, typename TIn>
struct VState {
    static constexpr int P = pow3(N - 1), C = 1 << (N - 1);
    int pm[P];
    int tlow[C];
    Raw<N> next;
    PlaneCursor<N, TIn> cur;
};

// In-plane box mins (3^(N-1) cells spanned by the vertex and its in-plane
// neighbours) from a plane's raw values: x +- 1 by warp shuffles.
template <int N, int CONS, typename TIn>
__device__ __forceinline__ void plane_reduce(const Raw<N> &r, int (&o)[pow3(N - 1)]) {
    const int lane = threadIdx.x & 31;
    int v[Raw<N>::R * 3];
#pragma unroll
    for (int k = 0; k < Raw<N>::R; ++k) {
        const int l = __shfl_up_sync(0xffffffffu, r.m[k], 1), rr = __shfl_down_sync(0xffffffffu, r.m[k], 1);
        v[k * 3] = lane == 0 ? r.h[k] : l;
        v[k * 3 + 1] = r.m[k];
        v[k * 3 + 2] = lane == 31 ? r.h[k] : rr;
    }
    if constexpr (N == 3) {
#pragma unroll
        for (int dx = 0; dx < 3; ++dx) {  // y pass: cells spanned by y and y + o_y
            v[dx] = min(v[dx], v[3 + dx]);
            v[6 + dx] = min(v[6 + dx], v[3 + dx]);
        }
    }
#pragma unroll
    for (int dy = 0; dy < Raw<N>::R; ++dy) {  // x pass
        v[dy * 3] = min(v[dy * 3], v[dy * 3 + 1]);
        v[dy * 3 + 2] = min(v[dy * 3 + 2], v[dy * 3 + 1]);
    }
#pragma unroll
    for (int i = 0; i < pow3(N - 1); ++i) {
        if constexpr (CONS == EUCALC_VERTEX && sizeof(TIn) == 1) o[i] = max(v[i], 0);  // mask commutes with min
        else o[i] = v[i];
    }
}

template <int N, int CONS, typename TIn>
__device__ __forceinline__ void masked_ie(const int (&in)[pow3(N - 1)], int (&t)[1 << (N - 1)]) {
    int v[pow3(N - 1)];
#pragma unroll
    for (int i = 0; i < pow3(N - 1); ++i) {
        if constexpr (CONS == EUCALC_VERTEX && sizeof(TIn) == 1) v[i] = in[i];  // masked in plane_boxmin
        else v[i] = mask_cell<CONS, TIn>(in[i]);
    }
    incl_excl<N - 1>(v);
#pragma unroll
    for (int c = 0; c < (1 << (N - 1)); ++c) t[c] = v[corner<N - 1>(c)];
}

// Prime the walk at plane w: pm = box mins of w, tlow = corners of min(w-1, w),
// plane w+1 in flight.
template <int N, int CONS, typename TIn>
__device__ __forceinline__ void vwalk_prime(const TIn *img, const Geo &g, int w, int y, int x, VState<N, TIn> &s) {
    constexpr int S = Sent<CONS, TIn>::value;
    Raw<N> r0, r1;
    s.cur.init(img, g, w - 1, y, x);
    s.cur.load(S, r0);
    s.cur.load(S, r1);
    s.cur.load(S, s.next);
    int pp[pow3(N - 1)];
    plane_reduce<N, CONS, TIn>(r0, pp);
    plane_reduce<N, CONS, TIn>(r1, s.pm);
#pragma unroll
    for (int i = 0; i < pow3(N - 1); ++i) pp[i] = min(pp[i], s.pm[i]);
    masked_ie<N, CONS, TIn>(pp, s.tlow);
}

// One walk step: Delta^- of all 2^N sign vectors at plane w, state advanced to w + 1.
// Orthant e: bit 0 <-> the walk axis (axis 0), bit k <-> axis k.
template <int N, int CONS, typename TIn>
__device__ __forceinline__ void vwalk_step(VState<N, TIn> &s, int (&dm)[1 << N]) {
    constexpr int P = pow3(N - 1), C = 1 << (N - 1);
    int pn[P], cu[P], tup[C], tmid[C];
    Raw<N> ahead;
    s.cur.load(Sent<CONS, TIn>::value, ahead);  // plane w + 2, in flight during this step
    plane_reduce<N, CONS, TIn>(s.next, pn);
#pragma unroll
    for (int i = 0; i < P; ++i) cu[i] = min(s.pm[i], pn[i]);  // cells spanning w .. w+1
    masked_ie<N, CONS, TIn>(cu, tup);
    masked_ie<N, CONS, TIn>(s.pm, tmid);
    static_for<0, (1 << N)>([&](auto E) {
        constexpr int e = decltype(E)::value;
        // in-plane bits: axis k (k >= 1) <-> bit k of e <-> corner bit j = k - 1 (slowest first)
        constexpr int c = e >> 1;
        if constexpr (e & 1) dm[e] = tmid[c] - s.tlow[c];
        else dm[e] = tmid[c] - tup[c];
    });
#pragma unroll
    for (int c = 0; c < C; ++c) s.tlow[c] = tup[c];
#pragma unroll
    for (int i = 0; i < P; ++i) s.pm[i] = pn[i];
    s.next = ahead;
}

// ------------------------------------------------------------------ TOP walk
// The vertex's 2^N pixels (bit k of the corner set <-> pixel x_k, clear <-> x_k - 1);
// the walk carries the pixels of plane w - 1 (bit 0 clear).
template <int N>
struct TState {
    int prev[1 << (N - 1)];
};

template <int N, typename TIn>
__device__ __forceinline__ void top_plane(const TIn *img, const Geo &g, int p, int y, int x, int (&o)[1 << (N - 1)]) {
    // pixels (p, y-1 / y, x-1 / x) of plane p; in-plane corner bit 0 <-> axis 1, ...
    constexpr int S = Sent<EUCALC_TOP, TIn>::value;
    const bool pok = p >= 0 && p < (N == 3 ? g.mZ : g.mY);
    int dummy;
    if constexpr (N == 3) {
#pragma unroll
        for (int by = 0; by < 2; ++by) {
            const int yy = y - 1 + by;
            const bool ok = pok && yy >= 0 && yy < g.mY;
            int l, m;
            load_row<TIn, false>(img + ((long long)p * g.mY + (ok ? yy : 0)) * g.mX, ok, x, g.mX, S, l, m, dummy);
            o[by * 2 + 0] = l;  // bit for axis 2 (x) is the low bit of the in-plane index
            o[by * 2 + 1] = m;
        }
    } else {
        int l, m;
        load_row<TIn, false>(img + (long long)(pok ? p : 0) * g.mX, pok, x, g.mX, S, l, m, dummy);
        o[0] = l;
        o[1] = m;
    }
}

template <int N, typename TIn>
__device__ __forceinline__ void twalk_step(const TIn *img, const Geo &g, int w, int y, int x, TState<N> &s,
                                           int (&dm)[1 << N]) {
    constexpr int P3 = pow3(N), PX = 1 << N;
    int cur[1 << (N - 1)];
    top_plane<N, TIn>(img, g, w, y, x, cur);
    // pix[c]: c bit k (axis k) set <-> pixel index x_k; in-plane index of axes 1..N-1
    // has axis N-1 (x) as its lowest bit
    int pix[PX];
    static_for<0, PX>([&](auto CC) {
        constexpr int c = decltype(CC)::value;
        constexpr int ip = N == 3 ? (((c >> 1) & 1) << 1) | ((c >> 2) & 1) : ((c >> 1) & 1);
        if constexpr (c & 1) pix[c] = cur[ip];
        else pix[c] = s.prev[ip];
    });
    int val[P3];
    static_for<0, P3>([&](auto I) {
        constexpr int idx = decltype(I)::value;
        int m = INT_MAX;
        static_for<0, PX>([&](auto C) {
            if constexpr (top_coface<N>(idx, decltype(C)::value)) m = min(m, pix[decltype(C)::value]);
        });
        val[idx] = mask_cell<EUCALC_TOP, TIn>(m);
    });
    incl_excl<N>(val);
    static_for<0, PX>([&](auto E) {
        constexpr int e = decltype(E)::value;
        constexpr int idx = (e & 1 ? 2 * pow3(N - 1) : 0) + ((e >> 1) & 1 ? 2 * pow3(N - 2) : 0) +
                            (N == 3 && ((e >> 2) & 1) ? 2 : 0);
        dm[e] = val[idx];
    });
#pragma unroll
    for (int i = 0; i < (1 << (N - 1)); ++i) s.prev[i] = cur[i];
}

// ------------------------------------------------------------------ the pencil kernel
template <int N, int CONS, typename TIn>
struct Walker {
    VState<N, TIn> v;
    TState<N> t;
    __device__ __forceinline__ void prime(const TIn *img, const Geo &g, int w, int y, int x) {
        if constexpr (CONS == EUCALC_VERTEX) vwalk_prime<N, CONS, TIn>(img, g, w, y, x, v);
        else top_plane<N, TIn>(img, g, w - 1, y, x, t.prev);
    }
    __device__ __forceinline__ void step(const TIn *img, const Geo &g, int w, int y, int x, int (&dm)[1 << N]) {
        if constexpr (CONS == EUCALC_VERTEX) vwalk_step<N, CONS, TIn>(v, dm);
        else twalk_step<N, TIn>(img, g, w, y, x, t, dm);
    }
};

// Predicated record store (no branch around it: a divergent `if` costs a
// reconvergence and the address setup on one side only).
__device__ __forceinline__ void st_rec_if(Rec16 *p, uint32_t c, int a, int b, bool pred) {
    const unsigned w = (unsigned)(a & 0xffff) | ((unsigned)b << 16);
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %3, 0;\n\t@q st.global.v2.b32 [%0], {%1, %2};\n\t}" ::"l"(p),
                 "r"(c), "r"(w), "r"((unsigned)pred)
                 : "memory");
}
__device__ __forceinline__ void st_rec_if(Rec32 *p, uint32_t c, int a, int b, bool pred) {
    if (pred) {
        p->c = c;
        p->a = a;
        p->b = b;
    }
}

// MODE kEmit : records into the (tile, warp) regions of the scratch lists, the
//              regions' counts and the |Delta^-| statistics of the lists;
//      kStats: per-orthant N^-, N^ord (eucalc_critical_counts).
template <int N, int CONS, typename TIn, typename RecT, int MODE>
__global__ void __launch_bounds__(kThreads, 3) k1_pencil(K1Args a) {
    constexpr int Q = 1 << (N - 1), FULL = (1 << N) - 1;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    Geo g;
    g.MX = a.M[N - 1];
    g.MY = N >= 2 ? a.M[N - 2] : 1;
    g.MZ = N == 3 ? a.M[0] : 1;
    g.mX = a.m[N - 1];
    g.mY = N >= 2 ? a.m[N - 2] : 1;
    g.mZ = N == 3 ? a.m[0] : 1;
    const int tiles_img = a.tiles_x * a.tiles_y * a.tiles_z;
    // this warp's pencil: image b, column block tx (x0 = 32 tx), row y (3-D) and
    // walk range [w0, w1) over the walk axis (z in 3-D, y in 2-D)
    long long b;
    int tx, y, w0, w1, ty_t, tz0, wslot;
    if constexpr (N == 3) {
        const int nzc = (g.MZ + kWalk3 - 1) / kWalk3;
        long long cta = blockIdx.x;
        tx = (int)(cta % a.tiles_x);
        cta /= a.tiles_x;
        ty_t = (int)(cta % a.tiles_y);
        cta /= a.tiles_y;
        const int zc = (int)(cta % nzc);
        b = cta / nzc;
        y = ty_t * Tile<N>::TY + warp;
        w0 = zc * kWalk3;
        w1 = min(g.MZ, w0 + kWalk3);
        tz0 = w0 / Tile<N>::TZ;
        wslot = warp;
        if (y >= g.MY) return;
    } else {
        const long long gw = (long long)blockIdx.x * kWarps + warp;
        if (gw >= a.batch * tiles_img * a.W) return;
        const int r = (int)(gw % a.W);
        b = gw / a.W / tiles_img;
        const int t = (int)(gw / a.W % tiles_img);
        tx = t % a.tiles_x;
        ty_t = t / a.tiles_x;
        y = 0;
        w0 = ty_t * Tile<N>::TY + r * (Tile<N>::TY / a.W);
        w1 = min(g.MY, w0 + Tile<N>::TY / a.W);
        tz0 = 0;
        wslot = r;
        if (w0 >= g.MY) return;  // an empty region of a ragged tile (its count stays 0)
    }
    const int x = tx * 32 + lane;
    const bool xin = x < g.MX;
    const TIn *img = reinterpret_cast<const TIn *>(a.img) + b * a.npix;
    const int W = N == 3 ? Tile<3>::W : a.W;  // warps (regions) per tile
    // records go to this (tile, warp)'s region of the scratch lists (fixed capacity
    // cap_r = its vertex count), or straight to the lists when an image is one region
    RecT *out = reinterpret_cast<RecT *>(a.direct ? a.rec : a.scratch);
    const long long lcap = a.direct ? a.vcap : a.scap;
    int run[Q];       // kept records so far in the current (tile, warp)
    RecT *dst[Q];     // first record of the current (tile, warp) region in each list
    using AccT = std::conditional_t<std::is_same<RecT, Rec16>::value, int, long long>;
    AccT abs_sum[Q];
    int max_rec[Q];
    int cnt_c[1 << N], cnt_o[Q];
#pragma unroll
    for (int q = 0; q < Q; ++q) {
        run[q] = 0;
        dst[q] = out;
        abs_sum[q] = 0;
        max_rec[q] = 0;
        cnt_o[q] = 0;
    }
#pragma unroll
    for (int e = 0; e < (1 << N); ++e) cnt_c[e] = 0;
    // the (tile, warp) slot of the tile holding walk step w
    auto slot = [&](int w) -> long long {
        const int tt = N == 3 ? ((tz0 + (w - w0) / Tile<N>::TZ) * a.tiles_y + ty_t) * a.tiles_x + tx
                              : ty_t * a.tiles_x + tx;
        return (long long)tt * W + wslot;
    };
    auto flush = [&](int w_last) {  // the (tile, warp) holding step w_last is complete
        if constexpr (MODE == kEmit) {
            if (lane == 0) {
                const long long sl = slot(w_last);
#pragma unroll
                for (int q = 0; q < Q; ++q) {
                    if (a.direct) {  // one region per image: its count is the list length
                        a.count[b * Q + q] = run[q];
                        a.tile_off[(b * Q + q) * 2] = 0;
                        a.tile_off[(b * Q + q) * 2 + 1] = run[q];
                    } else {
                        a.cnt[(b * Q + q) * (long long)tiles_img * W + sl] = run[q];
                    }
                }
            }
        }
#pragma unroll
        for (int q = 0; q < Q; ++q) run[q] = 0;
    };
    auto load_base = [&](int w) {
        if constexpr (MODE == kEmit) {
            const long long sl = slot(w);
#pragma unroll
            for (int q = 0; q < Q; ++q) dst[q] = out + (b * Q + q) * lcap + sl * a.cap_r;
        }
    };
    Walker<N, CONS, TIn> wk;
    wk.prime(img, g, w0, y, x);
    load_base(w0);
    const int seg = N == 3 ? Tile<3>::SEG : Tile<2>::TY / a.W;  // walk steps per region
    int left = seg;
    for (int w = w0; w < w1; ++w) {
        if (left == 0) {  // tile boundary
            flush(w - 1);
            load_base(w);
            left = seg;
        }
        --left;
        int dm[1 << N];
        wk.step(img, g, w, y, x, dm);
        if (!xin) {
#pragma unroll
            for (int e = 0; e < (1 << N); ++e) dm[e] = 0;
        }
        if constexpr (MODE == kStats) {
#pragma unroll
            for (int e = 0; e < (1 << N); ++e) cnt_c[e] += dm[e] != 0;
#pragma unroll
            for (int q = 0; q < Q; ++q) cnt_o[q] += dm[q] != dm[q ^ FULL];
        } else {
            uint32_t coord = 0;
            if constexpr (MODE == kEmit) {
                coord = (uint32_t)x << a.sh[N - 1];
                if constexpr (N == 3) coord |= ((uint32_t)y << a.sh[1]) | ((uint32_t)w << a.sh[0]);
                else coord |= (uint32_t)w << a.sh[0];
            }
#pragma unroll
            for (int q = 0; q < Q; ++q) {
                const int da = dm[q], db = dm[q ^ FULL];
                const bool keep = (da | db) != 0;
                const unsigned bal = __ballot_sync(0xffffffffu, keep);
                EU_DCHECK(!keep || run[q] + __popc(bal & ((1u << lane) - 1)) < (a.direct ? (int)a.vcap : a.cap_r));
                st_rec_if(dst[q] + run[q] + __popc(bal & ((1u << lane) - 1)), coord, da, db, keep);
                const int s = abs(da) + abs(db);
                abs_sum[q] += s;
                max_rec[q] = max(max_rec[q], s);
                run[q] += __popc(bal);
            }
        }
    }
    flush(w1 - 1);
    if constexpr (MODE == kEmit) {
        // |Delta^-| statistics of the lists (order-independent integer reductions)
#pragma unroll
        for (int q = 0; q < Q; ++q) {
            AccT v = abs_sum[q];
            for (int d = 16; d; d >>= 1) v += __shfl_xor_sync(0xffffffffu, v, d);
            if (lane == 0 && v) atomicAdd((unsigned long long *)&a.abs_sum[b * Q + q], (unsigned long long)(long long)v);
            int mr = max_rec[q];
            for (int d = 16; d; d >>= 1) mr = max(mr, __shfl_xor_sync(0xffffffffu, mr, d));
            if (lane == 0 && mr) atomicMax((unsigned long long *)&a.max_rec[b * Q + q], (unsigned long long)mr);
        }
    }
    if constexpr (MODE == kStats) {
#pragma unroll
        for (int e = 0; e < (1 << N); ++e) {
            int c = cnt_c[e], o = cnt_o[(e >> (N - 1)) & 1 ? (e ^ FULL) : e];
            for (int d = 16; d; d >>= 1) {
                c += __shfl_xor_sync(0xffffffffu, c, d);
                o += __shfl_xor_sync(0xffffffffu, o, d);
            }
            if (lane == 0) {
                if (c) atomicAdd((unsigned long long *)&a.stats[(b * (1 << N) + e) * 2], (unsigned long long)c);
                if (o) atomicAdd((unsigned long long *)&a.stats[(b * (1 << N) + e) * 2 + 1], (unsigned long long)o);
            }
        }
    }
}

// ------------------------------------------------------------------ 3-D VERTEX 8-bit: two vertices per lane
// For 8-bit VERTEX images a missing vertex can carry the sentinel 0 instead of
// -1: the masked cell value max(min(..., -1), 0) = 0 = min(..., 0) and every
// real value is >= 0. Masking then disappears and every box min is a plain min
// of values in [0, 255], so a lane can hold the columns x0 = 64 tx + 2 lane and
// x0 + 1 as the two 16-bit halves of one register: the mins run as one
// VIMNMX.U16x2 for both vertices, and the inclusion-exclusion subtractions as
// one IADD3 each (a + K - b) with a bias K per level that keeps both halves
// non-negative, so no borrow crosses from the low half into the high half:
//   box mins            [0, 255]            bias 0
//   x pass  v(0)-v(+-1) |.| <= 255          bias 256  (K1)
//   y pass  (corners)   |.| <= 510          bias 512  (K2)
//   Delta^- (walk axis) |.| <= 1020         bias 1024 (K3)
// (each level's K exceeds the previous level's range, so every half stays in
// [0, 2044]). The result is the same Delta^- as the scalar walk above, bit for
// bit; only the arithmetic is packed. A warp covers 64 columns, so the tiles of
// this variant are 64 x 8 x 8 vertices (k1_geometry).
namespace v8 {
constexpr uint32_t K1 = 0x01000100u, K2 = 0x02000200u, K3 = 0x04000400u, K4 = 0x08000800u;
constexpr uint32_t kUnbias = 0xfc00fc00u;  // -1024 in each half (VIADD.16x2)

__device__ __forceinline__ uint32_t mn(uint32_t a, uint32_t b) { return __vminu2(a, b); }

// predicated loads (no branch, nothing dereferenced when !ok): a u16 pair of
// columns, or one byte
__device__ __forceinline__ uint32_t ld_u16(const uint8_t *p, bool ok) {
    uint32_t v;
    asm("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\tmov.u32 %0, 0;\n\t@q ld.global.nc.u16 %0, [%1];\n\t}"
        : "=r"(v) : "l"(p), "r"((unsigned)ok));
    return v;
}
__device__ __forceinline__ uint32_t ld_u8(const uint8_t *p, bool ok) {
    uint32_t v;
    asm("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\tmov.u32 %0, 0;\n\t@q ld.global.nc.u8 %0, [%1];\n\t}"
        : "=r"(v) : "l"(p), "r"((unsigned)ok));
    return v;
}

// One plane's raw values for a lane: rows y-1, y, y+1 as packed column pairs
// (low half x0, high half x0+1) and the halo column (lane 0: x0-1 in the high
// half, lane 31: x0+2 in the low half; 0 elsewhere).
struct Raw {
    uint32_t m[3], h[3];
};

// Loads of consecutive planes (AL: rows start on even addresses, so a column
// pair is one u16 load). Lane pointers are fixed (row y-1, column x0, and the
// halo column); the plane offset and the row stride are CTA-uniform, so the
// per-step address arithmetic runs on the uniform datapath.
template <bool AL>
struct Cursor {
    const uint8_t *bp, *hp;  // lane's (row y-1, column x0) and halo column of plane 0
    long long po, pstride;   // uniform: offset of the next plane to load
    int rstride, p, pend, hsh;
    unsigned rmask;          // bit k: row y-1+k exists
    bool ok0, ok1, hok;
    __device__ __forceinline__ void init(const uint8_t *img, int MX, int MY, int MZ, int p0, int y, int x0) {
        const int lane = threadIdx.x & 31;
        const int hdx = lane == 0 ? -1 : 2;
        hsh = lane == 0 ? 16 : 0;
        ok0 = x0 < MX;
        ok1 = x0 + 1 < MX;
        hok = (lane == 0 || lane == 31) && (unsigned)(x0 + hdx) < (unsigned)MX;
        pstride = (long long)MY * MX;
        rstride = MX;
        p = p0;
        pend = MZ;
        rmask = 0;
        for (int k = 0; k < 3; ++k) rmask |= ((unsigned)(y - 1 + k) < (unsigned)MY ? 1u : 0u) << k;
        bp = img + (long long)(y - 1) * MX + x0;
        hp = bp + hdx;
        po = (long long)p0 * pstride;
    }
    __device__ __forceinline__ void load(Raw &r) {
        const bool pok = (unsigned)p < (unsigned)pend;
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            const long long o = po + (long long)k * rstride;
            const bool ok = pok && ((rmask >> k) & 1u);
            if constexpr (AL) {
                // bytes b0 b1 -> halves (b0, b1)
                r.m[k] = __byte_perm(ld_u16(bp + o, ok && ok0), 0u, 0x4140);
            } else {
                r.m[k] = __byte_perm(ld_u8(bp + o, ok && ok0), ld_u8(bp + o + 1, ok && ok1), 0x5410);
            }
            r.h[k] = ld_u8(hp + o, ok && hok) << hsh;
        }
        po += pstride;
        ++p;
    }
};

// In-plane box mins of the 3 x 3 cells around both vertices (index dy * 3 + dx,
// digit 0 <-> offset -1): x +- 1 by warp shuffles and byte permutes.
__device__ __forceinline__ void plane_reduce(const Raw &r, uint32_t (&o)[9]) {
    const int lane = threadIdx.x & 31;
    uint32_t A[3][3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const uint32_t M = r.m[k];
        uint32_t up = __shfl_up_sync(0xffffffffu, M, 1), dn = __shfl_down_sync(0xffffffffu, M, 1);
        up = lane == 0 ? r.h[k] : up;   // high half: column x0 - 1
        dn = lane == 31 ? r.h[k] : dn;  // low half: column x0 + 2
        const uint32_t L = __byte_perm(up, M, 0x5432);  // (x0-1, x0)
        const uint32_t R = __byte_perm(M, dn, 0x5432);  // (x0+1, x0+2)
        A[k][0] = mn(L, M);
        A[k][1] = M;
        A[k][2] = mn(M, R);
    }
#pragma unroll
    for (int dx = 0; dx < 3; ++dx) {
        o[dx] = mn(A[0][dx], A[1][dx]);
        o[3 + dx] = A[1][dx];
        o[6 + dx] = mn(A[2][dx], A[1][dx]);
    }
}

// In-plane inclusion-exclusion to the 4 corners (bit 0 <-> y, bit 1 <-> x; set
// <-> +1), bias 512 (10 IADD3).
__device__ __forceinline__ void ie(const uint32_t (&v)[9], uint32_t (&t)[4]) {
    uint32_t xp[3], xm[3];
#pragma unroll
    for (int r = 0; r < 3; ++r) {
        xp[r] = v[r * 3 + 1] + K1 - v[r * 3 + 0];  // slot +1: v(0) - v(-1)
        xm[r] = v[r * 3 + 1] + K1 - v[r * 3 + 2];  // slot -1: v(0) - v(+1)
    }
    t[0] = xm[1] + K2 - xm[2];  // y -1, x -1
    t[1] = xm[1] + K2 - xm[0];  // y +1, x -1
    t[2] = xp[1] + K2 - xp[2];  // y -1, x +1
    t[3] = xp[1] + K2 - xp[0];  // y +1, x +1
}

// Walk state at plane w
struct State {
    uint32_t pm[9];    // box mins of plane w
    uint32_t tlow[4];  // corners of min(plane w-1, plane w)
    uint32_t tmid[4];  // corners of plane w
    Raw next;          // raw plane w+1 (loaded one step ahead)
};

template <bool AL>
__device__ __forceinline__ void prime(Cursor<AL> &cur, State &s, const uint8_t *img, int MX, int MY, int MZ, int w,
                                      int y, int x0) {
    Raw r0, r1;
    cur.init(img, MX, MY, MZ, w - 1, y, x0);
    cur.load(r0);
    cur.load(r1);
    cur.load(s.next);
    uint32_t pp[9];
    plane_reduce(r0, pp);
    plane_reduce(r1, s.pm);
#pragma unroll
    for (int i = 0; i < 9; ++i) pp[i] = mn(pp[i], s.pm[i]);
    ie(pp, s.tlow);
    ie(s.pm, s.tmid);
}

// Delta^- + 1024 of both vertices for all 8 sign vectors at plane w (e bit 0
// <-> z, bit 1 <-> y, bit 2 <-> x) from the state `in` at w; `out` = the state
// at w + 1 (two states alternate, so advancing costs no register moves)
template <bool AL>
__device__ __forceinline__ void step(Cursor<AL> &cur, const State &in, State &out, uint32_t (&dm)[8]) {
    cur.load(out.next);  // plane w + 2, in flight during this step and the next
    uint32_t cu[9];
    plane_reduce(in.next, out.pm);
#pragma unroll
    for (int i = 0; i < 9; ++i) cu[i] = mn(in.pm[i], out.pm[i]);
    ie(cu, out.tlow);
    ie(out.pm, out.tmid);
#pragma unroll
    for (int e = 0; e < 8; ++e) {
        const int c = e >> 1;
        dm[e] = (e & 1) ? in.tmid[c] + K3 - in.tlow[c] : in.tmid[c] + K3 - out.tlow[c];
    }
}

__device__ __forceinline__ void st_rec_w(Rec16 *p, uint32_t c, uint32_t w, bool pred) {
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %3, 0;\n\t@q st.global.v2.b32 [%0], {%1, %2};\n\t}" ::"l"(p),
                 "r"(c), "r"(w), "r"((unsigned)pred)
                 : "memory");
}
}  // namespace v8

// Records of a 3-D 8-bit VERTEX image into the (tile, warp) regions (as
// k1_pencil<3, VERTEX, uint8_t, Rec16, kEmit>, tiles 64 x 8 x 8, a.walk planes per
// CTA). Region order: walk step, lane, column (x0 before x0 + 1).
template <bool AL>
__global__ void __launch_bounds__(kThreads, 3) k1_pencil_v8(K1Args a) {
    constexpr int Q = 4, TZ = 8;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int MX = a.M[2], MY = a.M[1], MZ = a.M[0];
    const int tiles_img = a.tiles_x * a.tiles_y * a.tiles_z;
    const int nzc = (MZ + a.walk - 1) / a.walk;
    long long cta = blockIdx.x;
    const int tx = (int)(cta % a.tiles_x);
    cta /= a.tiles_x;
    const int ty_t = (int)(cta % a.tiles_y);
    cta /= a.tiles_y;
    const int zc = (int)(cta % nzc);
    const long long b = cta / nzc;
    const int y = ty_t * 8 + warp;
    if (y >= MY) return;
    const int w0 = zc * a.walk, w1 = min(MZ, w0 + a.walk), tz0 = w0 / TZ;
    const int x0 = tx * 64 + 2 * lane;
    const uint8_t *img = reinterpret_cast<const uint8_t *>(a.img) + b * a.npix;
    Rec16 *out = reinterpret_cast<Rec16 *>(a.direct ? a.rec : a.scratch);
    const long long lcap = a.direct ? a.vcap : a.scap;
    int run[Q];
    Rec16 *dst[Q];
#pragma unroll
    for (int q = 0; q < Q; ++q) run[q] = 0;
    auto slot = [&](int w) -> long long {
        const int tt = ((tz0 + (w - w0) / TZ) * a.tiles_y + ty_t) * a.tiles_x + tx;
        return (long long)tt * 8 + warp;
    };
    auto load_base = [&](int w) {
        const long long sl = slot(w);
#pragma unroll
        for (int q = 0; q < Q; ++q) dst[q] = out + (b * Q + q) * lcap + sl * a.cap_r;
    };
    auto flush = [&](int w_last) {
        if (lane == 0) {
            const long long sl = slot(w_last);
#pragma unroll
            for (int q = 0; q < Q; ++q) {
                if (a.direct) {
                    a.count[b * Q + q] = run[q];
                    a.tile_off[(b * Q + q) * 2] = 0;
                    a.tile_off[(b * Q + q) * 2 + 1] = run[q];
                } else {
                    a.cnt[(b * Q + q) * (long long)tiles_img * 8 + sl] = run[q];
                }
            }
        }
#pragma unroll
        for (int q = 0; q < Q; ++q) run[q] = 0;
    };
    v8::Cursor<AL> cur;
    v8::State sa, sb;
    v8::prime(cur, sa, img, MX, MY, MZ, w0, y, x0);
    load_base(w0);
    const uint32_t cstep = 1u << a.sh[2];
    uint32_t coord = ((uint32_t)x0 << a.sh[2]) | ((uint32_t)y << a.sh[1]) | ((uint32_t)w0 << a.sh[0]);
    const uint32_t cw = 1u << a.sh[0];
    const unsigned lt = (1u << lane) - 1;
    // the |Delta^-| statistics of the lists are taken by k1_copy (it reads every record)
    auto emit = [&](const uint32_t (&dm)[8]) {
#pragma unroll
        for (int q = 0; q < Q; ++q) {
            const uint32_t r0 = __vadd2(__byte_perm(dm[q], dm[q ^ 7], 0x5410), v8::kUnbias);  // x0: a | b << 16
            const uint32_t r1 = __vadd2(__byte_perm(dm[q], dm[q ^ 7], 0x7632), v8::kUnbias);  // x0 + 1
            const bool k0 = r0 != 0, k1 = r1 != 0;
            const unsigned b0 = __ballot_sync(0xffffffffu, k0), b1 = __ballot_sync(0xffffffffu, k1);
            if ((b0 | b1) == 0) continue;  // nothing kept by the warp (most steps of binary images)
            const int p0 = run[q] + __popc(b0 & lt) + __popc(b1 & lt);
            EU_DCHECK(p0 + (int)k0 + (int)k1 <= a.cap_r || (a.direct && p0 + 2 <= a.vcap));
            v8::st_rec_w(dst[q] + p0, coord, r0, k0);
            v8::st_rec_w(dst[q] + p0 + (int)k0, coord + cstep, r1, k1);
            run[q] += __popc(b0) + __popc(b1);
        }
        coord += cw;
    };
    // two walk steps per iteration (states a -> b -> a); regions are 8 planes and
    // start on even steps, so a region boundary falls between iterations
    int w = w0;
    for (; w + 1 < w1; w += 2) {
        if (w > w0 && ((w - w0) & (TZ - 1)) == 0) {  // tile boundary
            flush(w - 1);
            load_base(w);
        }
        uint32_t dm[8];
        v8::step(cur, sa, sb, dm);
        emit(dm);
        v8::step(cur, sb, sa, dm);
        emit(dm);
    }
    if (w < w1) {  // odd tail
        if (w > w0 && ((w - w0) & (TZ - 1)) == 0) {
            flush(w - 1);
            load_base(w);
        }
        uint32_t dm[8];
        v8::step(cur, sa, sb, dm);
        emit(dm);
    }
    flush(w1 - 1);
}

// Exclusive scan of each list's (tile, warp) counts, in place -> offsets; the
// per-tile offsets (first warp of each tile) and the list length. One warp per
// chunk of 256 counts, chunks handed out by a ticket in list order; a chunk's
// prefix comes from a warp-wide decoupled look-back over the earlier chunks of
// its list (flag = status in bits 62-63: 1 aggregate, 2 inclusive prefix).
constexpr int kScanPer = 8, kScanChunk = 32 * kScanPer;
constexpr unsigned long long kAgg = 1ull << 62, kIncl = 2ull << 62, kValMask = (1ull << 62) - 1;

__device__ __forceinline__ unsigned long long ld_relaxed(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_relaxed(unsigned long long *p, unsigned long long v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__global__ void __launch_bounds__(kThreads) k1_scan(K1Args a, long long chunks_per_list, long long total) {
    const int lane = threadIdx.x & 31;
    unsigned tk = 0;
    if (lane == 0) tk = atomicAdd(a.ticket, 1u);
    tk = __shfl_sync(0xffffffffu, tk, 0);
    if (tk >= total) return;
    const long long L = tk / chunks_per_list, j = tk % chunks_per_list;
    const int tiles_img = a.tiles_x * a.tiles_y * a.tiles_z;
    const long long n = (long long)tiles_img * a.W;
    int32_t *c = a.cnt + L * n;
    const long long i0 = j * kScanChunk + (long long)lane * kScanPer;
    int v[kScanPer];
    int t = 0;
#pragma unroll
    for (int k = 0; k < kScanPer; ++k) {
        v[k] = i0 + k < n ? c[i0 + k] : 0;
        t += v[k];
    }
    int incl = t;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const int u = __shfl_up_sync(0xffffffffu, incl, d);
        if (lane >= d) incl += u;
    }
    const long long agg = __shfl_sync(0xffffffffu, incl, 31);
    unsigned long long *flag = a.flags + tk;
    long long prefix = 0;
    if (j == 0) {
        if (lane == 0) st_relaxed(flag, kIncl | (unsigned long long)agg);
    } else {
        if (lane == 0) st_relaxed(flag, kAgg | (unsigned long long)agg);
        long long back = j - 1;  // predecessor chunks j-1 .. 0 of this list (flags tk-1 .. tk-j)
        while (true) {
            const long long idx = back - lane;
            unsigned long long f = kIncl;  // virtual inclusive 0 before chunk 0
            if (idx >= 0) {
                const unsigned long long *p = a.flags + (tk - j + idx);
                do { f = ld_relaxed(p); } while ((f >> 62) == 0);
            }
            const unsigned inc = __ballot_sync(0xffffffffu, (f >> 62) == 2);
            const int first = inc ? __ffs(inc) - 1 : 31;
            long long val = lane <= first ? (long long)(f & kValMask) : 0;
            for (int d = 16; d; d >>= 1) val += __shfl_xor_sync(0xffffffffu, val, d);
            prefix += val;
            if (inc) break;
            back -= 32;
        }
        if (lane == 0) st_relaxed(flag, kIncl | (unsigned long long)(prefix + agg));
    }
    long long run = prefix + incl - t;
    int32_t *toff = a.tile_off + L * (long long)(tiles_img + 1);
#pragma unroll
    for (int k = 0; k < kScanPer; ++k) {
        const long long i = i0 + k;
        if (i < n) {
            c[i] = (int32_t)run;
            if (i % a.W == 0) toff[i / a.W] = (int32_t)run;
        }
        run += v[k];
    }
    if (j == chunks_per_list - 1 && lane == 0) {
        toff[tiles_img] = (int32_t)(prefix + agg);
        a.count[L] = (int32_t)(prefix + agg);
    }
}

// The records of every (tile, warp) region, from its fixed-capacity scratch
// region to its scanned position. A CTA owns kCopyRegions consecutive regions of
// a list; each warp copies whole regions (lanes over the region's records, four
// records in flight per lane): coalesced loads and stores, no per-record search.
constexpr int kCopyRegions = 32;

template <typename RecT>
__global__ void __launch_bounds__(kThreads) k1_copy(K1Args a, long long cpl) {
    __shared__ int s_off[kCopyRegions + 1];
    const long long L = blockIdx.x / cpl, j = blockIdx.x % cpl;
    const long long nreg = (long long)a.tiles_x * a.tiles_y * a.tiles_z * a.W;
    const long long r0 = j * kCopyRegions;
    const int nr = (int)min((long long)kCopyRegions, nreg - r0);
    const int32_t *off = a.cnt + L * nreg + r0;
    for (int i = threadIdx.x; i < nr; i += kThreads) s_off[i] = off[i];
    if (threadIdx.x == 0) s_off[nr] = r0 + nr < nreg ? off[nr] : a.count[L];
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const RecT *src0 = reinterpret_cast<const RecT *>(a.scratch) + L * a.scap + r0 * a.cap_r;
    RecT *dst0 = reinterpret_cast<RecT *>(a.rec) + L * a.vcap;
    long long ssum = 0;
    int smax = 0;
    auto stat = [&](const RecT &r) {
        if (a.stats_in_copy) {
            const int v = abs((int)r.a) + abs((int)r.b);
            ssum += v;
            smax = max(smax, v);
        }
    };
    constexpr int U = 4;
    // Two regions per warp step, all loads of a step issued before its stores and the
    // ragged ends predicated: a region holds ~100 records of a gray volume and ~15 of a
    // binary one, so a scalar tail loop would serialise load -> store round trips.
    for (int r = warp; r < nr; r += 2 * kWarps) {
        const int r2 = r + kWarps;
        const int c1 = s_off[r + 1] - s_off[r], c2 = r2 < nr ? s_off[r2 + 1] - s_off[r2] : 0;
        EU_DCHECK(c1 >= 0 && c1 <= a.cap_r && s_off[r] + c1 <= a.vcap);
        EU_DCHECK(c2 >= 0 && c2 <= a.cap_r && (r2 >= nr || s_off[r2] + c2 <= a.vcap));
        const RecT *src1 = src0 + (long long)r * a.cap_r, *src2 = src0 + (long long)r2 * a.cap_r;
        RecT *dst1 = dst0 + s_off[r], *dst2 = dst0 + (r2 < nr ? s_off[r2] : 0);
        const int cm = max(c1, c2);
        for (int i = lane; i < cm; i += U * 32) {
            RecT v1[U], v2[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                if (i + u * 32 < c1) v1[u] = src1[i + u * 32];
                if (i + u * 32 < c2) v2[u] = src2[i + u * 32];
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                if (i + u * 32 < c1) {
                    dst1[i + u * 32] = v1[u];
                    stat(v1[u]);
                }
                if (i + u * 32 < c2) {
                    dst2[i + u * 32] = v2[u];
                    stat(v2[u]);
                }
            }
        }
    }
    if (a.stats_in_copy) {  // |Delta^-| statistics of the list (order-independent integer reductions)
        __shared__ long long s_sum[kWarps];
        __shared__ int s_max[kWarps];
        for (int k = 16; k; k >>= 1) {
            ssum += __shfl_xor_sync(0xffffffffu, ssum, k);
            smax = max(smax, __shfl_xor_sync(0xffffffffu, smax, k));
        }
        if (lane == 0) {
            s_sum[warp] = ssum;
            s_max[warp] = smax;
        }
        __syncthreads();
        if (threadIdx.x == 0) {  // one atomic per CTA and statistic
            for (int w = 1; w < kWarps; ++w) {
                ssum += s_sum[w];
                smax = max(smax, s_max[w]);
            }
            if (ssum) atomicAdd((unsigned long long *)&a.abs_sum[L], (unsigned long long)ssum);
            if (smax) atomicMax((unsigned long long *)&a.max_rec[L], (unsigned long long)smax);
        }
    }
}

template <int N, int CONS, typename TIn, typename RecT>
cudaError_t launch_t(const K1Args &a, cudaStream_t s, int mode) {
    const int tiles_img = a.tiles_x * a.tiles_y * a.tiles_z;
    long long grid;
    if (N == 3) {
        const int nzc = (a.M[0] + kWalk3 - 1) / kWalk3;
        grid = a.batch * (long long)a.tiles_x * a.tiles_y * nzc;
    } else {
        grid = (a.batch * tiles_img * a.W + kWarps - 1) / kWarps;
    }
    if (grid == 0) return cudaSuccess;
    if (mode == kStats) {
        k1_pencil<N, CONS, TIn, RecT, kStats><<<(unsigned)grid, kThreads, 0, s>>>(a);
        count_launch();
        return cudaGetLastError();
    }
    k1_pencil<N, CONS, TIn, RecT, kEmit><<<(unsigned)grid, kThreads, 0, s>>>(a);
    count_launch();
    if (a.direct) return cudaGetLastError();  // one region per image: written in place
    const long long cpl = ((long long)tiles_img * a.W + kScanChunk - 1) / kScanChunk;
    const long long chunks = a.batch * (1 << (N - 1)) * cpl;
    k1_scan<<<(unsigned)((chunks + kWarps - 1) / kWarps), kThreads, 0, s>>>(a, cpl, chunks);
    const long long ccpl = ((long long)tiles_img * a.W + kCopyRegions - 1) / kCopyRegions;
    k1_copy<RecT><<<(unsigned)(a.batch * (1 << (N - 1)) * ccpl), kThreads, 0, s>>>(a, ccpl);
    count_launch(2);
    return cudaGetLastError();
}

template <int N, int CONS, typename TIn>
cudaError_t launch_r(const K1Args &a, cudaStream_t s, int mode) {
    return a.wide ? launch_t<N, CONS, TIn, Rec32>(a, s, mode) : launch_t<N, CONS, TIn, Rec16>(a, s, mode);
}

// 3-D 8-bit VERTEX images: the two-vertices-per-lane pencils, then the same scan
// and copy as launch_t
cudaError_t launch_v8(const K1Args &a, cudaStream_t s) {
    const int tiles_img = a.tiles_x * a.tiles_y * a.tiles_z;
    const int nzc = (a.M[0] + a.walk - 1) / a.walk;
    const long long grid = a.batch * (long long)a.tiles_x * a.tiles_y * nzc;
    if (grid == 0) return cudaSuccess;
    if (a.M[2] % 2 == 0) k1_pencil_v8<true><<<(unsigned)grid, kThreads, 0, s>>>(a);
    else k1_pencil_v8<false><<<(unsigned)grid, kThreads, 0, s>>>(a);
    count_launch();
    if (a.direct) return cudaGetLastError();
    const long long cpl = ((long long)tiles_img * a.W + kScanChunk - 1) / kScanChunk;
    const long long chunks = a.batch * 4 * cpl;
    k1_scan<<<(unsigned)((chunks + kWarps - 1) / kWarps), kThreads, 0, s>>>(a, cpl, chunks);
    const long long ccpl = ((long long)tiles_img * a.W + kCopyRegions - 1) / kCopyRegions;
    k1_copy<Rec16><<<(unsigned)(a.batch * 4 * ccpl), kThreads, 0, s>>>(a, ccpl);
    count_launch(2);
    return cudaGetLastError();
}
bool use_v8(const K1Args &a) { return a.TX == 64; }
template <int N, int CONS>
cudaError_t launch_d(const K1Args &a, cudaStream_t s, int mode) {
    switch (a.dtype) {
    case EUCALC_U8: return launch_r<N, CONS, uint8_t>(a, s, mode);
    case EUCALC_I16: return launch_r<N, CONS, int16_t>(a, s, mode);
    default: return launch_r<N, CONS, int32_t>(a, s, mode);
    }
}
cudaError_t launch_any(const K1Args &a_in, cudaStream_t s, int mode) {
    if (use_v8(a_in)) {
        if (mode == kEmit) {
            K1Args a = a_in;
            a.stats_in_copy = true;
            return launch_v8(a, s);
        }
    }
    K1Args a = a_in;
    if (a.ndim == 3 && a.TX != 32) {  // the scalar kernel's statistics pass over 32-wide column blocks
        a.TX = 32;
        a.tiles_x = (a.M[2] + 31) / 32;
    }
    if (a.ndim == 2)
        return a.construction == EUCALC_VERTEX ? launch_d<2, EUCALC_VERTEX>(a, s, mode)
                                               : launch_d<2, EUCALC_TOP>(a, s, mode);
    return a.construction == EUCALC_VERTEX ? launch_d<3, EUCALC_VERTEX>(a, s, mode)
                                           : launch_d<3, EUCALC_TOP>(a, s, mode);
}

}  // namespace

int64_t k1_scan_chunks(int64_t lists, int64_t ntiles, int W) {
    return lists * ((ntiles * W + kScanChunk - 1) / kScanChunk);
}

int k1_walk(int ndim, const int64_t *M, int64_t batch, int TX, int TY) {
    if (ndim != 3) return 0;
    // planes per CTA: long walks amortise the 2-plane prime, but keep >= 6 CTAs per SM's worth of work
    const int64_t cols = batch * ((M[2] + TX - 1) / TX) * ((M[1] + TY - 1) / TY);
    int walk = 64;
    while (walk > 8 && cols * ((M[0] + walk - 1) / walk) < 6 * 148) walk /= 2;
    return walk;
}

void k1_geometry(int ndim, const int64_t *M, int dtype, int construction, int *TX, int *TY, int *TZ, int *W) {
    *TX = 32;
    if (ndim == 3) {
        // 8-bit VERTEX volumes: two vertices per lane (k1_pencil_v8), 64-wide tiles
        if (dtype == EUCALC_U8 && construction == EUCALC_VERTEX && !getenv("EUCALC_K1_SCALAR")) *TX = 64;
        *TY = 8;
        *TZ = 8;
        *W = 8;
    } else {
        *TY = 64;
        *TZ = 1;
        *W = (M[1] <= 32 && M[0] <= 64) ? 1 : 4;
    }
}

cudaError_t launch_k1(const K1Args &a, cudaStream_t s) { return launch_any(a, s, kEmit); }
cudaError_t launch_k1_stats(const K1Args &a, cudaStream_t s) { return launch_any(a, s, kStats); }

}  // namespace eucalc
