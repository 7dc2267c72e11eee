// K1 — critical points (SURVEY 8(a) A1 stencil + A2 ordered compaction).
//
// For every vertex x of every image and every sign vector eps:
//   Delta^-(eps, x) = chi(phi | lwst(eps, x))
// where the lower star is the set of cells at doubled coordinates 2x - delta o eps,
// delta in {0,1}^n, restricted to existing cells (E16). One CTA owns a
// tile of vertices (full rows when they fit, so lists come out in row-major
// vertex order); the image tile plus a one-vertex halo is staged in shared
// memory as int32 with a sentinel for out-of-range positions:
//   VERTEX: phi(cell) = min of its vertices; out-of-range vertex = INT_MIN,
//                   so a cell touching it has phi = INT_MIN = "does not exist".
//   TOP: phi(cell) = min over its top cofaces (pixels); out-of-range
//                   pixel = INT_MAX, so a cell whose fixed pixel index is out of
//                   range has phi = INT_MAX = "does not exist", while an in-range
//                   face at the image border takes the min of its real cofaces.
// Per vertex all 3^n star-cell values are formed in registers (separable mins),
// masked to 0 where the cell does not exist, and the 2^n lower-star sums come
// from an in-register inclusion-exclusion transform (38 adds in 3-D).
//
// Compaction: per antipodal pair {eps, -eps} (eps the representative with
// eps_{n-1} = -1) a vertex is kept iff Delta^-(eps) != 0 or Delta^-(-eps) != 0
// (this covers the classical points of both orthants and every ordinary point,
// since J(eps) = Delta^-(eps) - Delta^-(-eps)). Warp ballot/popc + block scan
// give the in-tile order; a decoupled look-back over the image's tiles (dynamic
// ticket order) gives each tile's global offset, so the list order is
// deterministic (tile-major; within a tile by warp, vertex batch and lane) with
// a single pass.
// Tiles are boxes of <= kTileV vertices (the whole image when it fits; else
// 64 x 32 in 2-D, 16 x 16 x 8 in 3-D), so a tile spans a narrow band of heights
// in every direction; K1 records each tile's list offset for K2's culling.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>

#include <climits>
#include <type_traits>

#include "eucalc_internal.cuh"

namespace eucalc {
namespace {

constexpr int kThreads = 256;
constexpr int kTileV = 2048;  // vertices per tile (max)
constexpr int kPerWarp = kTileV / (kThreads / 32);  // staging slice per warp

__host__ __device__ constexpr int pow3(int k) { return k == 0 ? 1 : 3 * pow3(k - 1); }

template <typename T>
__device__ __forceinline__ int load_img(const T *p, int64_t i) { return (int)__ldg(p + i); }

__device__ __forceinline__ unsigned long long ld_relaxed(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_relaxed(unsigned long long *p, unsigned long long v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// Flag word for the tile look-back: status in bits 62..63 (1 = aggregate,
// 2 = inclusive prefix), count in the low 62 bits.
constexpr unsigned long long kAgg = 1ull << 62, kIncl = 2ull << 62, kValMask = (1ull << 62) - 1;

// Warp-wide decoupled look-back. Returns the exclusive prefix of tile `t`
// (t >= 1) given flags for tiles [0, t) of this (image, pair); `stride` between
// consecutive tiles' flag words.
__device__ long long lookback(unsigned long long *flag_t, int t, int stride, long long agg) {
    const int lane = threadIdx.x & 31;
    long long excl = 0;  // the tile's aggregate is already published (k1_tile)
    int j = t - 1;
    while (true) {
        int idx = j - lane;
        unsigned long long f = kIncl;  // virtual inclusive 0 before tile 0
        if (idx >= 0) {
            const unsigned long long *p = flag_t - (long long)(t - idx) * stride;
            do { f = ld_relaxed(p); } while ((f >> 62) == 0);
        }
        unsigned incl = __ballot_sync(0xffffffffu, (f >> 62) == 2);
        int first = incl ? __ffs(incl) - 1 : 31;
        long long v = (lane <= first) ? (long long)(f & kValMask) : 0;
        for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        excl += v;
        if (incl) break;
        j -= 32;
    }
    if (lane == 0) st_relaxed(flag_t, kIncl | (unsigned long long)(excl + agg));
    return excl;
}

// Compile-time loop: f(std::integral_constant<int, I>) for I in [B, E). Every
// index below is a constant expression, so the 3^n star values stay in
// registers (a runtime-indexed array would live in local memory).
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

// Staged region element: int16 for 8-bit images (the sentinels -32768 / 32767
// lie outside 0..255: half the shared memory, more CTAs per SM), else int32.
template <typename TIn>
using RegT = std::conditional_t<sizeof(TIn) == 1, short, int>;
template <typename R>
__host__ __device__ constexpr int sent_lo() { return sizeof(R) == 2 ? -32768 : INT_MIN; }
template <typename R>
__host__ __device__ constexpr int sent_hi() { return sizeof(R) == 2 ? 32767 : INT_MAX; }

template <int N, int CONS, typename R>
__device__ __forceinline__ void vertex_dminus(const R *s, int sz, int sy, int base, int (&dm)[1 << N]) {
    constexpr int P3 = pow3(N);
    int val[P3];
    auto stride = [&](int k) { return (k == N - 1) ? 1 : ((k == N - 2) ? sy : sz); };
    if constexpr (CONS == EUCALC_VERTEX) {
        // point values of the 3^n neighbourhood, then separable box mins: after
        // axis k, val[o] = min over the vertices of the cell spanned by x and x+o
        static_for<0, P3>([&](auto I) {
            constexpr int idx = decltype(I)::value;
            int off = 0;
            static_for<0, N>([&](auto K) { off += (digit3<N>(idx, decltype(K)::value) - 1) * stride(decltype(K)::value); });
            val[idx] = s[base + off];
        });
        static_for<0, N>([&](auto K) {
            constexpr int k = decltype(K)::value, st = pow3(N - 1 - k);
            static_for<0, P3>([&](auto I) {
                constexpr int idx = decltype(I)::value, ok = digit3<N>(idx, k);
                if constexpr (ok != 1) val[idx] = min(val[idx], val[idx + (1 - ok) * st]);
            });
        });
        static_for<0, P3>([&](auto I) {
            constexpr int idx = decltype(I)::value;
            // 8-bit images (int16 region): weights >= 0 > sentinel, so one max masks
            if constexpr (sizeof(R) == 2) val[idx] = max(val[idx], 0);
            else val[idx] = (val[idx] == sent_lo<R>()) ? 0 : val[idx];
        });
    } else {
        // 2^n pixels around the vertex (pixel x + c, c in {-1,0}^n); base <-> c = 0
        constexpr int P2 = 1 << N;
        int pix[P2];
        static_for<0, P2>([&](auto C) {
            constexpr int c = decltype(C)::value;
            int off = 0;
            static_for<0, N>([&](auto K) {
                if constexpr (!((c >> decltype(K)::value) & 1)) off -= stride(decltype(K)::value);
            });
            pix[c] = s[base + off];
        });
        static_for<0, P3>([&](auto I) {
            constexpr int idx = decltype(I)::value;
            int mval = sent_hi<R>();
            static_for<0, P2>([&](auto C) {
                if constexpr (top_coface<N>(idx, decltype(C)::value)) mval = min(mval, pix[decltype(C)::value]);
            });
            val[idx] = (mval == sent_hi<R>()) ? 0 : mval;
        });
    }
    // inclusion-exclusion: along axis k, slot +1 <- z(0) - z(-1) (eps_k=+1), slot -1 <- z(0) - z(+1)
    static_for<0, N>([&](auto K) {
        constexpr int k = decltype(K)::value, st = pow3(N - 1 - k);
        static_for<0, P3>([&](auto I) {
            constexpr int idx = decltype(I)::value;
            if constexpr (digit3<N>(idx, k) == 1) {
                const int a = val[idx - st], c = val[idx], b = val[idx + st];
                val[idx + st] = c - a;
                val[idx - st] = c - b;
            }
        });
    });
    static_for<0, (1 << N)>([&](auto E) {
        constexpr int e = decltype(E)::value;
        constexpr int idx = (((e >> 0) & 1) ? 2 * pow3(N - 1) : 0) + (N > 1 && ((e >> 1) & 1) ? 2 * pow3(N - 2) : 0) +
                            (N > 2 && ((e >> 2) & 1) ? 2 * pow3(N - 3 < 0 ? 0 : N - 3) : 0);
        dm[e] = val[idx];
    });
}

// ---- 3-D VERTEX, 8-bit region: a thread walks one z-column of the tile and
// carries the planes it shares with the next vertex. The box mins and the
// inclusion-exclusion above are separable (min and the per-axis difference
// commute), and max(min(a,b),0) = min(max(a,0),max(b,0)), so per vertex only the
// new plane z+1 is loaded, min-reduced in-plane and masked; the z pass combines
// planes. In-plane values p[dy*3+dx], digit 0/1/2 <-> offset -1/0/+1.
__device__ __forceinline__ void plane_min(const short *s, int sy, int pbase, int (&p)[9]) {
#pragma unroll
    for (int dy = 0; dy < 3; ++dy)
#pragma unroll
        for (int dx = 0; dx < 3; ++dx) p[dy * 3 + dx] = s[pbase + (dy - 1) * sy + (dx - 1)];
#pragma unroll
    for (int dx = 0; dx < 3; ++dx) {  // y pass: cells spanned by x and x + o_y
        p[dx] = min(p[dx], p[3 + dx]);
        p[6 + dx] = min(p[6 + dx], p[3 + dx]);
    }
#pragma unroll
    for (int dy = 0; dy < 3; ++dy) {  // x pass
        p[dy * 3] = min(p[dy * 3], p[dy * 3 + 1]);
        p[dy * 3 + 2] = min(p[dy * 3 + 2], p[dy * 3 + 1]);
    }
#pragma unroll
    for (int i = 0; i < 9; ++i) p[i] = max(p[i], 0);  // missing cell (sentinel) -> 0
}
// in-plane inclusion-exclusion, corner slots t[(dy>>1)*2 + (dx>>1)], dy, dx in {0,2}:
// slot 2 <- mid - (offset -1), slot 0 <- mid - (offset +1), as in vertex_dminus
__device__ __forceinline__ void plane_ie(const int (&p)[9], int (&t)[4]) {
    int r[3][2];
#pragma unroll
    for (int dy = 0; dy < 3; ++dy) {
        r[dy][1] = p[dy * 3 + 1] - p[dy * 3];
        r[dy][0] = p[dy * 3 + 1] - p[dy * 3 + 2];
    }
#pragma unroll
    for (int xs = 0; xs < 2; ++xs) {
        t[2 + xs] = r[1][xs] - r[0][xs];
        t[xs] = r[1][xs] - r[2][xs];
    }
}

// Shared state of one tile (per CTA).
template <int N>
struct K1Shared {
    int warp[kThreads / 32][1 << (N - 1)];
    int run[1 << (N - 1)];
    long long excl[1 << (N - 1)];
    int ostat[1 << N][2];
};

// One tile: stage the image region (from global memory, or from the raw TMA box
// `raw` of xbox x ybox x zbox elements at image coordinates (x0-xoff, y0-1, z0-1),
// xoff = 16 bytes of elements: TMA wants 16-byte aligned innermost box starts),
// run the stencil, compact, look back, copy out. All threads of the CTA call it;
// `sh.ostat` must be zero on entry (it is left zero on exit).
template <int N, int CONS, typename TIn, typename RecT>
__device__ __forceinline__ void k1_tile(const K1Args &a, unsigned ticket, const TIn *raw, int xbox, int ybox,
                                        RecT *stage, RegT<TIn> *reg, K1Shared<N> &sh) {
    constexpr int Q = 1 << (N - 1);
    constexpr int FULL = (1 << N) - 1;
    auto &s_warp = sh.warp;
    auto &s_run = sh.run;
    auto &s_excl = sh.excl;
    auto &s_ostat = sh.ostat;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int tiles_per_img = a.tiles_x * a.tiles_y * a.tiles_z;
    const int64_t b = ticket / tiles_per_img;
    const int t = ticket % tiles_per_img;
    const int tx = t % a.tiles_x, ty = (t / a.tiles_x) % a.tiles_y, tz = t / (a.tiles_x * a.tiles_y);

    // vertex-lattice extents along (z, y, x) view; a tile is a TZ x TY x TX box of vertices
    const int MX = a.M[N - 1];
    const int MY = (N >= 2) ? a.M[N - 2] : 1;
    const int MZ = (N == 3) ? a.M[0] : 1;
    const int mX = a.m[N - 1];
    const int mY = (N >= 2) ? a.m[N - 2] : 1;
    const int mZ = (N == 3) ? a.m[0] : 1;
    const int x0 = tx * a.TX, y0 = ty * a.TY, z0 = tz * a.TZ;
    const int TXe = min(a.TX, MX - x0), TYe = min(a.TY, MY - y0), TZe = (N == 3) ? min(a.TZ, MZ - z0) : 1;
    const int RX = TXe + 2, RY = TYe + 2, RZ = (N == 3) ? TZe + 2 : 1;

    // ---- stage the input region (image index = vertex idx for VERTEX, pixel idx
    // for TOP) with a one-voxel halo: planes z0-1 .. z0+TZe, rows y0-1 .. y0+TYe,
    // cols x0-1 .. x0+TXe; one warp per region row, lanes along the row
    const TIn *img = reinterpret_cast<const TIn *>(a.img) + b * a.npix;
    const int SENT = (CONS == EUCALC_VERTEX) ? sent_lo<RegT<TIn>>() : sent_hi<RegT<TIn>>();
    if (raw) {  // TMA box already in shared memory (out-of-range elements zero-filled)
        for (int row = warp; row < RZ * RY; row += kThreads / 32) {
            const int pz = row / RY, ry = row - pz * RY;
            const int gy = y0 - 1 + ry, gz = (N == 3) ? z0 - 1 + pz : 0;
            const bool rin = gy >= 0 && gy < mY && gz >= 0 && gz < mZ;
            RegT<TIn> *dst = reg + row * RX;
            const TIn *src = raw + ((long long)pz * ybox + ry) * xbox + (16 / (int)sizeof(TIn) - 1);
            for (int rx = lane; rx < RX; rx += 32) {
                const int gx = x0 - 1 + rx;
                dst[rx] = (rin && gx >= 0 && gx < mX) ? (int)src[rx] : SENT;
            }
        }
    } else {
        // flat walk over the region (all lanes busy), element index -> (pz, ry, rx)
        // advanced incrementally by kThreads (no division per element), four
        // (2-D) or eight (3-D: config 4 gray K1 0.390 -> 0.382 ms) loads in flight
        const int RXY = RX * RY, NR = RXY * RZ;
        const int sz_ = kThreads / RXY, r1 = kThreads - sz_ * RXY, sy_ = r1 / RX, sx_ = r1 - sy_ * RX;
        int pz = tid / RXY, rem = tid - pz * RXY, ry = rem / RX, rx = rem - ry * RX;
        constexpr int kLd = N == 3 ? 8 : 4;  // loads in flight per thread
        for (int i0 = tid; i0 < NR; i0 += kLd * kThreads) {
            int v[kLd];
#pragma unroll
            for (int u = 0; u < kLd; ++u) {
                const int gx = x0 - 1 + rx, gy = y0 - 1 + ry, gz = (N == 3) ? z0 - 1 + pz : 0;
                const bool in = i0 + u * kThreads < NR && gx >= 0 && gx < mX && gy >= 0 && gy < mY && gz >= 0 && gz < mZ;
                v[u] = in ? load_img(img, ((int64_t)gz * mY + gy) * mX + gx) : SENT;
                rx += sx_;
                if (rx >= RX) {
                    rx -= RX;
                    ++ry;
                }
                ry += sy_;
                if (ry >= RY) {
                    ry -= RY;
                    ++pz;
                }
                pz += sz_;
            }
#pragma unroll
            for (int u = 0; u < kLd; ++u)
                if (i0 + u * kThreads < NR) reg[i0 + u * kThreads] = v[u];
        }
    }
    __syncthreads();

    // ---- per vertex stencil + compaction into shared staging
    const int sy = RX, sz = RX * RY;
    const int TP = TXe * TYe;
    const int TV = TP * TZe;
    int cnt_o[1 << N][2];
#pragma unroll
    for (int e = 0; e < (1 << N); ++e) cnt_o[e][0] = cnt_o[e][1] = 0;
    // per thread: at most kTileV / kThreads vertices; 16-bit records keep the sum in int32
    using AccT = std::conditional_t<std::is_same<RecT, Rec16>::value, int, long long>;
    AccT abs_sum[Q];
    int max_rec[Q];
#pragma unroll
    for (int q = 0; q < Q; ++q) {
        abs_sum[q] = 0;
        max_rec[q] = 0;
    }

    int wrun[Q];
#pragma unroll
    for (int q = 0; q < Q; ++q) wrun[q] = 0;
    // vertex index li = c0 + tid -> (lz, ly, lx), advanced incrementally by kThreads
    const int vz_ = kThreads / TP, v1 = kThreads - vz_ * TP, vy_ = v1 / TXe, vx_ = v1 - vy_ * TXe;
    int lz = tid / TP, lrem = tid - lz * TP, ly = lrem / TXe, lx = lrem - ly * TXe;
    // full-plane tiles (TP == kThreads): vertex li + kThreads is the same (lx, ly) at lz + 1
    constexpr bool kSlide = N == 3 && CONS == EUCALC_VERTEX && sizeof(RegT<TIn>) == 2;
    const bool slide = kSlide && TP == kThreads;
    int sl_pm[9], sl_tlow[4];  // plane lz (masked box mins); corners of min(plane lz-1, plane lz)
    if constexpr (kSlide) {
        if (slide) {
            const int base0 = (lz + 1) * sz + (ly + 1) * sy + (lx + 1);
            int pp[9];
            plane_min(reinterpret_cast<const short *>(reg), sy, base0 - sz, pp);
            plane_min(reinterpret_cast<const short *>(reg), sy, base0, sl_pm);
#pragma unroll
            for (int i = 0; i < 9; ++i) pp[i] = min(pp[i], sl_pm[i]);
            plane_ie(pp, sl_tlow);
        }
    }
    for (int c0 = 0; c0 < TV; c0 += kThreads) {
        const int li = c0 + tid;
        const bool valid = li < TV;
        int dm[1 << N];
        if (kSlide && slide) {
            if constexpr (kSlide) {
                const int base = (lz + 1) * sz + (ly + 1) * sy + (lx + 1);
                int pn[9], cu[9], tup[4], tmid[4];
                plane_min(reinterpret_cast<const short *>(reg), sy, base + sz, pn);
#pragma unroll
                for (int i = 0; i < 9; ++i) cu[i] = min(sl_pm[i], pn[i]);  // cells spanning lz .. lz+1
                plane_ie(cu, tup);
                plane_ie(sl_pm, tmid);
                // z pass: slot 2 (eps_z = +1, bit 0 of e) <- mid - low, slot 0 <- mid - up
#pragma unroll
                for (int e = 0; e < (1 << N); ++e) {
                    const int i = ((e >> 1) & 1) * 2 + ((e >> 2) & 1);
                    dm[e] = (e & 1) ? tmid[i] - sl_tlow[i] : tmid[i] - tup[i];
                }
#pragma unroll
                for (int i = 0; i < 4; ++i) sl_tlow[i] = tup[i];
#pragma unroll
                for (int i = 0; i < 9; ++i) sl_pm[i] = pn[i];
            }
        } else if (valid) {
            const int base = ((N == 3) ? (lz + 1) * sz : 0) + (ly + 1) * sy + (lx + 1);
            vertex_dminus<N, CONS>(reg, sz, sy, base, dm);
        } else {
#pragma unroll
            for (int e = 0; e < (1 << N); ++e) dm[e] = 0;
        }
#pragma unroll
        for (int e = 0; e < (1 << N); ++e) {
            cnt_o[e][0] += dm[e] != 0;
            cnt_o[e][1] += dm[e] != dm[e ^ FULL];
        }
        uint32_t coord = 0;
        if (valid) {
            const int gx = x0 + lx, gy = y0 + ly;
            coord = ((uint32_t)gx << a.sh[N - 1]);
            if (N >= 2) coord |= ((uint32_t)gy << a.sh[N - 2]);
            if (N == 3) coord |= ((uint32_t)(z0 + lz) << a.sh[0]);
        }
        lx += vx_;
        if (lx >= TXe) {
            lx -= TXe;
            ++ly;
        }
        ly += vy_;
        if (ly >= TYe) {
            ly -= TYe;
            ++lz;
        }
        lz += vz_;
        // warp-private compaction: warp w appends to its own slice of the
        // staging area (no block barrier per vertex batch); the tile's order is
        // (warp, batch, lane) and the slices are concatenated at copy-out
#pragma unroll
        for (int q = 0; q < Q; ++q) {
            const bool keep = dm[q] != 0 || dm[q ^ FULL] != 0;
            const unsigned bal = __ballot_sync(0xffffffffu, keep);
            if (keep) {
                RecT r;
                r.c = coord;
                r.a = dm[q];
                r.b = dm[q ^ FULL];
                stage[q * kTileV + warp * kPerWarp + wrun[q] + __popc(bal & ((1u << lane) - 1))] = r;
            }
            wrun[q] += __popc(bal);
            abs_sum[q] += abs(dm[q]) + abs(dm[q ^ FULL]);
            max_rec[q] = max(max_rec[q], abs(dm[q]) + abs(dm[q ^ FULL]));
        }
    }
    if (lane == 0) {
#pragma unroll
        for (int q = 0; q < Q; ++q) s_warp[warp][q] = wrun[q];
    }
    __syncthreads();
    if (tid < Q) {
        int tot = 0;
        for (int w = 0; w < kThreads / 32; ++w) tot += s_warp[w][tid];
        s_run[tid] = tot;
        // publish this tile's aggregate now, before the statistics below, so that
        // successors looking back find it sooner (tile 0 publishes its inclusive prefix)
        unsigned long long *flag_t = a.flags + ((int64_t)b * tiles_per_img + t) * Q + tid;
        st_relaxed(flag_t, (t == 0 ? kIncl : kAgg) | (unsigned long long)tot);
    }

    // ---- per-image statistics (order-independent integer sums: deterministic)
#pragma unroll
    for (int e = 0; e < (1 << N); ++e) {
        int c = cnt_o[e][0], o = cnt_o[e][1];
        for (int d = 16; d; d >>= 1) {
            c += __shfl_xor_sync(0xffffffffu, c, d);
            o += __shfl_xor_sync(0xffffffffu, o, d);
        }
        if (lane == 0) {
            atomicAdd(&s_ostat[e][0], c);
            atomicAdd(&s_ostat[e][1], o);
        }
    }
#pragma unroll
    for (int q = 0; q < Q; ++q) {
        AccT v = abs_sum[q];
        for (int d = 16; d; d >>= 1) v += __shfl_xor_sync(0xffffffffu, v, d);
        if (lane == 0 && v) atomicAdd((unsigned long long *)&a.abs_sum[b * Q + q], (unsigned long long)(long long)v);
        int mr = max_rec[q];
        for (int d = 16; d; d >>= 1) mr = max(mr, __shfl_xor_sync(0xffffffffu, mr, d));
        if (lane == 0 && mr) atomicMax((unsigned long long *)&a.max_rec[b * Q + q], (unsigned long long)mr);
    }
    __syncthreads();
    if (tid < (1 << N) * 2) {
        int v = (&s_ostat[0][0])[tid];
        if (v) atomicAdd((unsigned long long *)&a.stats[b * (1 << N) * 2 + tid], (unsigned long long)v);
        (&s_ostat[0][0])[tid] = 0;  // ready for the CTA's next tile
    }

    // ---- look-back per pair (warp q), then ordered copy-out
    if (warp < Q) {
        const int q = warp;
        const long long agg = s_run[q];
        unsigned long long *flag_t = a.flags + ((int64_t)b * tiles_per_img + t) * Q + q;
        long long excl;
        if (t == 0) {
            excl = 0;  // inclusive prefix published with the aggregate
        } else {
            excl = lookback(flag_t, t, Q, agg);
        }
        if (lane == 0) {
            s_excl[q] = excl;
            // per-tile list offsets: K2's height-window culling streams only the
            // tiles whose height range meets the window
            int32_t *toff = a.tile_off + (b * Q + q) * (int64_t)(tiles_per_img + 1);
            toff[t] = (int32_t)excl;
            if (t == tiles_per_img - 1) {
                a.count[b * Q + q] = (int32_t)(excl + agg);
                toff[tiles_per_img] = (int32_t)(excl + agg);
            }
        }
    }
    __syncthreads();
    RecT *out = reinterpret_cast<RecT *>(a.rec);
#pragma unroll
    for (int q = 0; q < Q; ++q) {
        int before = 0;  // this warp's slice follows the slices of warps 0..warp-1
        for (int w = 0; w < warp; ++w) before += s_warp[w][q];
        RecT *dst = out + (b * Q + q) * a.vcap + s_excl[q] + before;
        const RecT *src = stage + q * kTileV + warp * kPerWarp;
        for (int i = lane; i < s_warp[warp][q]; i += 32) dst[i] = src[i];
    }
    __syncthreads();  // staging, region and shared counters are reused by the next tile
}

// 3-D: at most 80 registers so that three CTAs fit per SM (the 8-bit region +
// staging of a 16x16x8 tile is 72 KB, three fit in shared memory too)
template <int N, int CONS, typename TIn, typename RecT>
__global__ void __launch_bounds__(kThreads, N == 3 ? 3 : 1) k1_kernel(K1Args a) {
    constexpr int Q = 1 << (N - 1);
    extern __shared__ __align__(16) unsigned char smem[];
    RecT *stage = reinterpret_cast<RecT *>(smem);           // [Q][kTileV]
    RegT<TIn> *reg = reinterpret_cast<RegT<TIn> *>(stage + Q * kTileV);  // input region
    __shared__ K1Shared<N> sh;
    __shared__ unsigned s_ticket;
    if (threadIdx.x == 0) s_ticket = atomicAdd(a.ticket, 1u);
    if (threadIdx.x < (1 << N) * 2) (&sh.ostat[0][0])[threadIdx.x] = 0;
    __syncthreads();
    k1_tile<N, CONS, TIn, RecT>(a, s_ticket, nullptr, 0, 0, stage, reg, sh);
}

// ---- TMA-staged K1 for large images: a persistent CTA keeps the next tile's
// box (image region + halo) in flight with cp.async.bulk.tensor while it works
// on the current one (double buffer, one mbarrier per buffer). Requires 16-byte
// aligned image rows; the tensor map is 3-D (x, y, image) or 4-D (x, y, z, image).
__device__ __forceinline__ uint32_t smem_addr(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int N>
__device__ __forceinline__ void tma_box(const CUtensorMap *tm, void *dst, unsigned long long *bar, int x, int y, int z,
                                        int b) {
    if (N == 2)
        asm volatile(
            "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
            ::"r"(smem_addr(dst)), "l"(tm), "r"(x), "r"(y), "r"(b), "r"(smem_addr(bar))
            : "memory");
    else
        asm volatile(
            "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], "
            "[%6];" ::"r"(smem_addr(dst)),
            "l"(tm), "r"(x), "r"(y), "r"(z), "r"(b), "r"(smem_addr(bar))
            : "memory");
}

template <int N, int CONS, typename TIn, typename RecT>
__global__ void __launch_bounds__(kThreads) k1_tma(const __grid_constant__ CUtensorMap tm, K1Args a, int xbox, int ybox,
                                                   int zbox) {
    constexpr int Q = 1 << (N - 1);
    extern __shared__ __align__(128) unsigned char k1_smem_tma[];
    const int box_bytes = xbox * ybox * zbox * (int)sizeof(TIn);
    const int box_pad = (box_bytes + 127) / 128 * 128;
    TIn *raw[2] = {reinterpret_cast<TIn *>(k1_smem_tma), reinterpret_cast<TIn *>(k1_smem_tma + box_pad)};
    RecT *stage = reinterpret_cast<RecT *>(k1_smem_tma + 2 * box_pad);  // [Q][kTileV]
    RegT<TIn> *reg = reinterpret_cast<RegT<TIn> *>(stage + Q * kTileV);  // input region
    __shared__ K1Shared<N> sh;
    __shared__ unsigned long long bar[2];
    __shared__ unsigned s_next;
    const int tiles_per_img = a.tiles_x * a.tiles_y * a.tiles_z;
    const unsigned total = (unsigned)(a.batch * tiles_per_img);
    auto issue = [&](unsigned tk, int buf) {  // thread 0: TMA of tile tk's box into raw[buf]
        const int b = (int)(tk / tiles_per_img), t = (int)(tk % tiles_per_img);
        const int tx = t % a.tiles_x, ty = (t / a.tiles_x) % a.tiles_y, tz = t / (a.tiles_x * a.tiles_y);
        asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(&bar[buf])),
                     "r"(box_bytes)
                     : "memory");
        tma_box<N>(&tm, raw[buf], &bar[buf], tx * a.TX - 16 / (int)sizeof(TIn), ty * a.TY - 1, N == 3 ? tz * a.TZ - 1 : 0, b);
    };
    if (threadIdx.x == 0) {
        for (int k = 0; k < 2; ++k)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(&bar[k])) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        s_next = atomicAdd(a.ticket, 1u);
        if (s_next < total) issue(s_next, 0);
    }
    if (threadIdx.x < (1 << N) * 2) (&sh.ostat[0][0])[threadIdx.x] = 0;
    __syncthreads();
    unsigned cur = s_next;
    int buf = 0;
    unsigned phase[2] = {0, 0};
    while (cur < total) {
        __syncthreads();  // every thread has read s_next
        if (threadIdx.x == 0) {
            s_next = atomicAdd(a.ticket, 1u);
            if (s_next < total) issue(s_next, buf ^ 1);  // raw[buf^1] was consumed by the previous tile
        }
        // wait for this tile's box
        asm volatile(
            "{\n\t.reg .pred p;\nK1W_%=:\n\t"
            "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%0], %1;\n\t"
            "@!p bra K1W_%=;\n}" ::"r"(smem_addr(&bar[buf])),
            "r"(phase[buf])
            : "memory");
        phase[buf] ^= 1;
        k1_tile<N, CONS, TIn, RecT>(a, cur, raw[buf], xbox, ybox, stage, reg, sh);  // ends with __syncthreads
        cur = s_next;
        buf ^= 1;
    }
}


// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda)
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static bool tried = false;
    if (!tried) {
        tried = true;
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
        cudaGetLastError();
    }
    return fn;
}

template <typename TIn>
CUtensorMapDataType tma_type() {
    return sizeof(TIn) == 1 ? CU_TENSOR_MAP_DATA_TYPE_UINT8
                            : sizeof(TIn) == 2 ? CU_TENSOR_MAP_DATA_TYPE_UINT16 : CU_TENSOR_MAP_DATA_TYPE_INT32;
}

template <int N, int CONS, typename TIn, typename RecT>
cudaError_t launch_t(const K1Args &a, cudaStream_t s) {
    constexpr int Q = 1 << (N - 1);
    const int planes = (N == 3) ? a.TZ + 2 : 1;
    const size_t region = sizeof(RegT<TIn>) * planes * (a.TY + 2) * (a.TX + 2);
    const size_t stage = sizeof(RecT) * Q * kTileV;
    const int64_t ntiles = a.batch * (int64_t)a.tiles_x * a.tiles_y * a.tiles_z;
    // TMA path: tiled images with 16-byte aligned base, rows and tile origins, boxes
    // within 256 per dimension. The innermost box start must be 16-byte aligned
    // (measured: other starts fault), so a box spans cols x0-xoff .. x0+TX rounded
    // up to xoff, xoff = 16 bytes of elements, instead of the one-column halo.
    const int e = (int)sizeof(TIn), xoff = 16 / e;
    const int xbox = (xoff + a.TX + 1 + xoff - 1) / xoff * xoff, ybox = a.TY + 2, zbox = N == 3 ? a.TZ + 2 : 1;
    const bool tma = ntiles > 1 && ((int64_t)a.m[N - 1] * e) % 16 == 0 && (a.TX * e) % 16 == 0 &&
                     ((uintptr_t)a.img & 15) == 0 && xbox <= 256 && ybox <= 256 && zbox <= 256 &&
                     encode_fn() != nullptr && a.use_tma;
    if (tma) {
        CUtensorMap tm;
        cuuint64_t dims[5], strides[4];
        cuuint32_t box[5], estr[5] = {1, 1, 1, 1, 1};
        int rank = 0;
        dims[rank] = (cuuint64_t)a.m[N - 1];
        box[rank++] = (cuuint32_t)xbox;
        dims[rank] = (cuuint64_t)a.m[N - 2];
        box[rank++] = (cuuint32_t)ybox;
        if (N == 3) {
            dims[rank] = (cuuint64_t)a.m[0];
            box[rank++] = (cuuint32_t)zbox;
        }
        dims[rank] = (cuuint64_t)a.batch;
        box[rank++] = 1;
        cuuint64_t st = (cuuint64_t)a.m[N - 1] * e;
        for (int k = 0; k < rank - 1; ++k) {
            strides[k] = st;
            st *= dims[k + 1];
        }
        CUresult r = encode_fn()(&tm, tma_type<TIn>(), (cuuint32_t)rank, const_cast<void *>(a.img), dims, strides, box,
                                 estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                 CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r == CUDA_SUCCESS) {
            const size_t box_pad = ((size_t)xbox * ybox * zbox * e + 127) / 128 * 128;
            const size_t smem = 2 * box_pad + stage + region;
            auto kern = k1_tma<N, CONS, TIn, RecT>;
            int occ = 0;
            cudaError_t err = prepare_kernel((const void *)kern, kThreads, smem, &occ);
            if (err != cudaSuccess) return err;
            int dev = 0, sms = 148;
            cudaGetDevice(&dev);
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
            const int64_t grid = std::min<int64_t>(ntiles, (int64_t)std::max(occ, 1) * sms);
            kern<<<(unsigned)grid, kThreads, smem, s>>>(tm, a, xbox, ybox, zbox);
            count_launch();
            return cudaGetLastError();
        }
    }
    const size_t smem = stage + region;
    auto kern = k1_kernel<N, CONS, TIn, RecT>;
    cudaError_t err = prepare_kernel((const void *)kern, kThreads, smem, nullptr);
    if (err != cudaSuccess) return err;
    kern<<<(unsigned)ntiles, kThreads, smem, s>>>(a);
    count_launch();
    return cudaGetLastError();
}

template <int N, int CONS, typename TIn>
cudaError_t launch_r(const K1Args &a, cudaStream_t s) {
    return a.wide ? launch_t<N, CONS, TIn, Rec32>(a, s) : launch_t<N, CONS, TIn, Rec16>(a, s);
}
template <int N, int CONS>
cudaError_t launch_d(const K1Args &a, cudaStream_t s) {
    switch (a.dtype) {
    case EUCALC_U8: return launch_r<N, CONS, uint8_t>(a, s);
    case EUCALC_I16: return launch_r<N, CONS, int16_t>(a, s);
    default: return launch_r<N, CONS, int32_t>(a, s);
    }
}

}  // namespace

cudaError_t launch_k1(const K1Args &a, cudaStream_t s) {
    if (a.ndim == 2)
        return a.construction == EUCALC_VERTEX ? launch_d<2, EUCALC_VERTEX>(a, s) : launch_d<2, EUCALC_TOP>(a, s);
    return a.construction == EUCALC_VERTEX ? launch_d<3, EUCALC_VERTEX>(a, s) : launch_d<3, EUCALC_TOP>(a, s);
}

int k1_tile_vertices() { return kTileV; }

}  // namespace eucalc
