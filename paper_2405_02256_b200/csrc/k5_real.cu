// K5 — exact ECT / Radon for REAL-valued directions (NEXT row f3; the paper's
// experimental setting, directions drawn in [0,1]^n).
//
// Heights are no longer integers in a known range, so the counting sort of K2
// does not apply; this is the paper's own algorithm: per (image,
// direction) the critical records of the direction's orthant get their dot
// products, are sorted, equal dots are merged and cumulative sums taken.
//   h(x) = <xi, x>,  x_i = p_i / (M_i - 1) - 0.5  (0 when M_i = 1),
// evaluated as ((xi_0 x_0 + xi_1 x_1) + xi_2 x_2) + 0.0 in IEEE double with
// round-to-nearest intrinsics (no contraction into FMAs), so equal heights are
// exactly the equal computed dots (E22).
//
// One warp per segment: records -> (order-preserving 64-bit key of h,
// Delta^-, J) in shared memory, a warp-synchronous bitonic sort, then a warp
// scan of (Delta^-, J) in height order; at the end of each run of equal keys
// the three canonical streams are emitted exactly as in K2 (E8: zero-net runs
// dropped). Two launches: count (entries per segment) -> CSR scan -> emit.
#include <climits>

#include "eucalc_internal.cuh"

namespace eucalc {
namespace {

constexpr int kThreads = 256;

__device__ __forceinline__ unsigned long long order_key(double h) {
    const unsigned long long u = (unsigned long long)__double_as_longlong(h);
    return (u >> 63) ? ~u : (u | (1ull << 63));
}
__device__ __forceinline__ double key_height(unsigned long long k) {
    const unsigned long long u = (k >> 63) ? (k & ~(1ull << 63)) : ~k;
    return __longlong_as_double((long long)u);
}

template <typename RecT>
__device__ __forceinline__ double real_height(const RecT &r, const K5Args &a, const double *xi) {
    double h = 0.0;
#pragma unroll
    for (int k = 0; k < kMaxN; ++k) {
        if (k < a.ndim) {
            const int p = (int)((r.c >> a.sh[k]) & a.msk[k]);
            double x = 0.0;
            if (a.M[k] > 1) x = __dsub_rn(__ddiv_rn((double)p, (double)(a.M[k] - 1)), 0.5);
            const double t = __dmul_rn(xi[k], x);
            h = (k == 0) ? t : __dadd_rn(h, t);
        }
    }
    return __dadd_rn(h, 0.0);
}

__device__ __forceinline__ long long warp_incl_scan64(long long v) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const long long t = __shfl_up_sync(0xffffffffu, v, d);
        if (lane >= d) v += t;
    }
    return v;
}

// One warp per segment (W warps per CTA, each with its own shared-memory
// arrays of npow2 entries): warp-synchronous bitonic sort, warp scans.
template <typename RecT, typename OutV, bool EMIT>
__global__ void __launch_bounds__(kThreads) k5_real(K5Args a, int wpb) {
    extern __shared__ __align__(16) unsigned char k5_smem[];
    const int N = a.npow2;  // padded sort length (power of two >= every list length)
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (warp >= wpb) return;
    unsigned char *base = k5_smem + (size_t)warp * N * 16;
    unsigned long long *key = reinterpret_cast<unsigned long long *>(base);
    // (Delta^-, J) per record; after the scan the same words hold the inclusive
    // prefix sums in height order (int32: |sums| <= list sum |a|+|b| < 2^31, host-checked)
    int *wc = reinterpret_cast<int *>(key + N);
    int *wj = wc + N;
    int *cc = wc, *cj = wj;
    const long long S = a.batch * a.D;
    for (long long s = (long long)blockIdx.x * wpb + warp; s < S; s += (long long)gridDim.x * wpb) {
        const long long b = s / a.D, d = s - b * a.D;
        const double xi[kMaxN] = {a.xi[d * a.ndim], a.ndim > 1 ? a.xi[d * a.ndim + 1] : 0.0,
                                  a.ndim > 2 ? a.xi[d * a.ndim + 2] : 0.0};
        const int q = a.q[d], sw = a.swap[d];
        const RecT *list = reinterpret_cast<const RecT *>(a.rec) + (b * a.Q + q) * a.vcap;
        const int n = a.count[b * a.Q + q];
        if (n > a.small_max) continue;  // bucketed path (k5b_*), warp-uniform
        int np = 32;  // this segment's sort length
        while (np < n) np <<= 1;
        for (int i = lane; i < np; i += 32) {
            if (i < n) {
                const RecT r = list[i];
                key[i] = order_key(real_height(r, a, xi));
                wc[i] = sw ? r.b : r.a;
                wj[i] = sw ? (r.b - r.a) : (r.a - r.b);
            } else {
                key[i] = ULLONG_MAX;  // padding sorts last and is never emitted
                wc[i] = wj[i] = 0;
            }
        }
        __syncwarp();
        // bitonic sort of (key, wc, wj), ascending keys
        for (int k = 2; k <= np; k <<= 1) {
            for (int j = k >> 1; j > 0; j >>= 1) {
                // pair t -> (i, i + j): insert a 0 bit at position log2(j); every lane busy
                for (int t = lane; t < (np >> 1); t += 32) {
                    const int i = ((t & ~(j - 1)) << 1) | (t & (j - 1)), p = i | j;
                    const bool up = (i & k) == 0;
                    const unsigned long long ki = key[i], kp = key[p];
                    if (up ? (ki > kp) : (ki < kp)) {
                        key[i] = kp;
                        key[p] = ki;
                        const int c0 = wc[i], j0 = wj[i];
                        wc[i] = wc[p];
                        wj[i] = wj[p];
                        wc[p] = c0;
                        wj[p] = j0;
                    }
                }
                __syncwarp();
            }
        }
        // warp scan of (Delta^-, J) in height order: lane owns [lane*pl, (lane+1)*pl)
        const int pl = np / 32;
        const int i0 = lane * pl, i1 = i0 + pl;
        long long lc = 0, lj = 0;
        for (int i = i0; i < i1; ++i) {
            lc += wc[i];
            lj += wj[i];
        }
        {
            long long xc = warp_incl_scan64(lc) - lc, xj = warp_incl_scan64(lj) - lj;
            for (int i = i0; i < i1; ++i) {
                xc += wc[i];
                xj += wj[i];
                cc[i] = (int)xc;  // in place: wc[i] was read above
                cj[i] = (int)xj;
            }
        }
        __syncwarp();
        // run ends: emit flags and values (a run's head is found by walking back; runs are short)
        int nc = 0, no = 0;
        for (int i = i0; i < i1; ++i) {
            const unsigned long long k = key[i];
            if (i >= n || (i + 1 < np && key[i + 1] == k)) continue;
            int h0 = i;
            while (h0 > 0 && key[h0 - 1] == k) --h0;
            const int bc = h0 ? cc[h0 - 1] : 0, bj = h0 ? cj[h0 - 1] : 0;
            nc += cc[i] != bc;
            no += cj[i] != bj;
        }
        const long long pc_incl = warp_incl_scan64(nc), po_incl = warp_incl_scan64(no);
        if (!EMIT) {
            if (lane == 31) {
                a.cnt_c[s] = (int)pc_incl;
                a.cnt_o[s] = (int)po_incl;
            }
        } else {
            long long pc = (a.do_ect ? a.ect.off[s] : a.do_cls ? a.cls.off[s] : 0) + pc_incl - nc;
            long long po = (a.do_ord ? a.ord.off[s] : 0) + po_incl - no;
            for (int i = i0; i < i1; ++i) {
                const unsigned long long k = key[i];
                if (i >= n || (i + 1 < np && key[i + 1] == k)) continue;
                int h0 = i;
                while (h0 > 0 && key[h0 - 1] == k) --h0;
                const int bc = h0 ? cc[h0 - 1] : 0, bj = h0 ? cj[h0 - 1] : 0;
                const double h = key_height(k);
                if (cc[i] != bc) {
                    // ECT value after h; classical Radon(h) = Radon(h-) + sum Delta^- at h
                    if (a.do_ect) {
                        reinterpret_cast<double *>(a.ect.h)[pc] = h;
                        reinterpret_cast<OutV *>(a.ect.v)[pc] = (OutV)cc[i];
                    }
                    if (a.do_cls) {
                        if (!a.cls_alias) reinterpret_cast<double *>(a.cls.h)[pc] = h;
                        reinterpret_cast<OutV *>(a.cls.v)[pc] = (OutV)(bj + (cc[i] - bc));
                    }
                    ++pc;
                }
                if (cj[i] != bj) {
                    if (a.do_ord) {
                        reinterpret_cast<double *>(a.ord.h)[po] = h;
                        reinterpret_cast<OutV *>(a.ord.v)[po] = (OutV)cj[i];
                    }
                    ++po;
                }
            }
        }
        __syncwarp();
    }
}

template <typename RecT>
cudaError_t launch_r(const K5Args &a, int phase, cudaStream_t s, int num_sms) {
    const size_t per_warp = (size_t)a.npow2 * 16;
    const int wpb = (int)std::max<size_t>(1, std::min<size_t>(kThreads / 32, (size_t)(64 * 1024) / per_warp));
    const size_t smem = per_warp * wpb;
    auto k = phase == 0 ? k5_real<RecT, int64_t, false> : k5_real<RecT, int64_t, true>;
    int occ = 0;
    cudaError_t e = prepare_kernel((const void *)k, wpb * 32, smem, &occ);
    if (e != cudaSuccess) return e;
    const long long S = a.batch * a.D;
    const long long grid = std::min<long long>((S + wpb - 1) / wpb, (long long)std::max(occ, 1) * num_sms);
    k<<<(unsigned)grid, wpb * 32, smem, s>>>(a, wpb);
    count_launch();
    return cudaGetLastError();
}

// ============================================================================
// Bucketed path for long lists (> small_max records): the paper's sort
// as a value-bucket pass + per-piece sorts.
//   k5b_bucket : one CTA per segment: bucket index of every record's height
//                (monotone in h, so equal heights share a bucket), smem
//                histogram, scan -> piece table, scatter {key, Delta^-, J}
//                to the segment's scratch, grouped by bucket;
//   k5b_sort   : pieces of more than kK5PieceMax records (height clusters):
//                one CTA each, bitonic tiles of 8192 in smem + merge-path passes;
//   k5b_piece  : one warp per piece: warp bitonic sort in smem (written back),
//                then a streaming run-length merge (counts and sums), and in
//                the emit pass the canonical entries at the piece's offset;
//   k5b_segscan: exclusive scan of the pieces' counts and sums per segment.
__device__ __forceinline__ uint4 pack_rec(unsigned long long k, int wc, int wj) {
    return make_uint4((unsigned)k, (unsigned)(k >> 32), (unsigned)wc, (unsigned)wj);
}
__device__ __forceinline__ unsigned long long rec_key(const uint4 &r) {
    return ((unsigned long long)r.y << 32) | r.x;
}

struct SegView {
    long long s, b, d;
    double xi[kMaxN];
    int q, sw, n;
};
__device__ __forceinline__ SegView seg_view(const K5Args &a, long long s) {
    SegView v;
    v.s = s;
    v.b = s / a.D;
    v.d = s - v.b * a.D;
#pragma unroll
    for (int k = 0; k < kMaxN; ++k) v.xi[k] = k < a.ndim ? a.xi[v.d * a.ndim + k] : 0.0;
    v.q = a.q[v.d];
    v.sw = a.swap[v.d];
    v.n = a.count[v.b * a.Q + v.q];
    return v;
}

// bucket of height h: floor((h - lo) * scale) clamped to [0, nb); every step is
// monotone in h, so h1 <= h2 implies bucket(h1) <= bucket(h2)
__device__ __forceinline__ int bucket_of(double h, double lo, double scale, int nb) {
    const double v = __dmul_rn(__dsub_rn(h, lo), scale);
    return v <= 0.0 ? 0 : (v >= (double)(nb - 1) ? nb - 1 : (int)v);
}

constexpr int kBigThreads = 1024;

// block-wide exclusive scan of NV ints per thread (thread order); returns totals
template <int NV>
__device__ __forceinline__ void block_excl_scan(int (&v)[NV], int (&tot)[NV]) {
    __shared__ int s_w[kBigThreads / 32][NV];
    __shared__ int s_tot[NV];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    int x[NV];
#pragma unroll
    for (int c = 0; c < NV; ++c) {
        x[c] = v[c];
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const int t = __shfl_up_sync(0xffffffffu, x[c], d);
            if (lane >= d) x[c] += t;
        }
        if (lane == 31) s_w[warp][c] = x[c];
    }
    __syncthreads();
    if (warp == 0) {
#pragma unroll
        for (int c = 0; c < NV; ++c) {
            const int w = lane < nw ? s_w[lane][c] : 0;
            int y = w;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const int t = __shfl_up_sync(0xffffffffu, y, d);
                if (lane >= d) y += t;
            }
            if (lane < nw) s_w[lane][c] = y - w;
            if (lane == 31) s_tot[c] = y;
        }
    }
    __syncthreads();
#pragma unroll
    for (int c = 0; c < NV; ++c) {
        v[c] = s_w[warp][c] + x[c] - v[c];
        tot[c] = s_tot[c];
    }
    __syncthreads();
}

template <typename RecT>
__global__ void __launch_bounds__(kBigThreads) k5b_bucket(K5Args a, K5Big g) {
    extern __shared__ unsigned k5b_hist[];
    const long long i = blockIdx.x;
    const SegView sv = seg_view(a, g.seg[i]);
    const RecT *list = reinterpret_cast<const RecT *>(a.rec) + (sv.b * a.Q + sv.q) * a.vcap;
    const int n = sv.n, nb = g.nb[i];
    const long long pb = g.pbase[i], sb = g.sbase[i];
    double half = 0.0;
#pragma unroll
    for (int k = 0; k < kMaxN; ++k)
        if (k < a.ndim && a.M[k] > 1) half += fabs(sv.xi[k]) * 0.5;
    const double lo = -half, scale = half > 0.0 ? (double)nb / (2.0 * half) : 0.0;
    for (int k = threadIdx.x; k < nb; k += blockDim.x) k5b_hist[k] = 0;
    __syncthreads();
    for (int r = threadIdx.x; r < n; r += blockDim.x)
        atomicAdd(&k5b_hist[bucket_of(real_height(list[r], a, sv.xi), lo, scale, nb)], 1u);
    __syncthreads();
    // pieces: thread t owns buckets [k0, k1)
    const int per = (nb + blockDim.x - 1) / blockDim.x;
    const int k0 = min(nb, (int)threadIdx.x * per), k1 = min(nb, k0 + per);
    int v[1] = {0}, tot[1];
    for (int k = k0; k < k1; ++k) v[0] += (int)k5b_hist[k];
    block_excl_scan<1>(v, tot);
    int ex = v[0];
    for (int k = k0; k < k1; ++k) {
        const int c = (int)k5b_hist[k];
        const long long p = pb + k;
        g.p_start[p] = sb + ex;
        g.p_len[p] = c;
        g.p_seg[p] = (int32_t)i;
        if (c > kK5PieceMax) {
            const unsigned o = atomicAdd(g.over, 1u);
            if (o < (unsigned)g.over_cap) g.over[2 + o] = (unsigned)p;
        }
        k5b_hist[k] = (unsigned)ex;  // scatter cursor
        ex += c;
    }
    __syncthreads();
    for (int r = threadIdx.x; r < n; r += blockDim.x) {
        const RecT rr = list[r];
        const double h = real_height(rr, a, sv.xi);
        const unsigned pos = atomicAdd(&k5b_hist[bucket_of(h, lo, scale, nb)], 1u);
        const int wc = sv.sw ? rr.b : rr.a, wj = sv.sw ? (rr.b - rr.a) : (rr.a - rr.b);
        g.scr[sb + pos] = pack_rec(order_key(h), wc, wj);
    }
}

constexpr int kSortTile = 8192;  // records per smem tile of the CTA sort (128 KB)

__global__ void __launch_bounds__(kBigThreads) k5b_sort(K5Big g) {
    extern __shared__ uint4 k5b_tile[];
    __shared__ unsigned s_t;
    const unsigned nover = min(g.over[0], (unsigned)g.over_cap);
    while (true) {
        if (threadIdx.x == 0) s_t = atomicAdd(g.over + 1, 1u);
        __syncthreads();
        const unsigned t = s_t;
        __syncthreads();
        if (t >= nover) break;
        const long long p = g.over[2 + t];
        const long long st = g.p_start[p];
        const int len = g.p_len[p];
        uint4 *A = g.scr + st, *B = g.tmp + st;
        for (int t0 = 0; t0 < len; t0 += kSortTile) {
            const int m = min(kSortTile, len - t0);
            int np = 2;
            while (np < m) np <<= 1;
            for (int i = threadIdx.x; i < np; i += blockDim.x)
                k5b_tile[i] = i < m ? A[t0 + i] : make_uint4(~0u, ~0u, 0u, 0u);
            __syncthreads();
            for (int k = 2; k <= np; k <<= 1)
                for (int j = k >> 1; j > 0; j >>= 1) {
                    for (int u = threadIdx.x; u < (np >> 1); u += blockDim.x) {
                        const int i = ((u & ~(j - 1)) << 1) | (u & (j - 1)), q = i | j;
                        const bool up = (i & k) == 0;
                        const uint4 x = k5b_tile[i], y = k5b_tile[q];
                        const unsigned long long kx = rec_key(x), ky = rec_key(y);
                        if (up ? (kx > ky) : (kx < ky)) {
                            k5b_tile[i] = y;
                            k5b_tile[q] = x;
                        }
                    }
                    __syncthreads();
                }
            for (int i = threadIdx.x; i < m; i += blockDim.x) A[t0 + i] = k5b_tile[i];
            __syncthreads();
        }
        // merge passes (merge path, 8 outputs per thread per step; ties keep A first)
        uint4 *src = A, *dst = B;
        for (int w = kSortTile; w < len; w <<= 1) {
            for (int base = 0; base < len; base += 2 * w) {
                const int na = min(w, len - base), nbb = max(0, min(w, len - base - w));
                const uint4 *a0 = src + base, *b0 = src + base + na;
                const int tot = na + nbb;
                for (int k0 = threadIdx.x * 8; k0 < tot; k0 += blockDim.x * 8) {
                    int lo = max(0, k0 - nbb), hi = min(k0, na);
                    while (lo < hi) {
                        const int mid = (lo + hi) >> 1;
                        if (rec_key(a0[mid]) <= rec_key(b0[k0 - mid - 1])) lo = mid + 1;
                        else hi = mid;
                    }
                    int ia = lo, ib = k0 - lo;
                    for (int o = 0; o < 8 && k0 + o < tot; ++o) {
                        const bool takeA = ib >= nbb || (ia < na && rec_key(a0[ia]) <= rec_key(b0[ib]));
                        dst[base + k0 + o] = takeA ? a0[ia++] : b0[ib++];
                    }
                }
            }
            __syncthreads();
            uint4 *x = src;
            src = dst;
            dst = x;
        }
        if (src != A) {
            for (int i = threadIdx.x; i < len; i += blockDim.x) A[i] = src[i];
            __syncthreads();
        }
    }
}

// Streaming run-length merge of a sorted piece P[0, len) by one warp: at the
// end of each run of equal keys the canonical entries (E8: zero-net runs
// dropped) with running sums starting at (ic, ij).
template <bool EMIT>
__device__ __forceinline__ void rle_piece(const K5Args &a, const uint4 *P, int len, int ic, int ij, long long pc,
                                          long long po, int &nc, int &no, int &sc, int &sj) {
    const int lane = threadIdx.x & 31;
    const unsigned lt = (1u << lane) - 1u;
    int cum_c = ic, cum_j = ij, end_c = ic, end_j = ij;
    nc = no = 0;
    for (int w = 0; w < len; w += 32) {
        const int i = w + lane;
        const bool valid = i < len;
        const uint4 r = valid ? P[i] : make_uint4(0u, 0u, 0u, 0u);
        const unsigned long long k = rec_key(r);
        unsigned long long kn = __shfl_down_sync(0xffffffffu, k, 1);
        if (lane == 31 && i + 1 < len) kn = rec_key(P[i + 1]);
        const bool is_end = valid && (i + 1 == len || kn != k);
        int xc = valid ? (int)r.z : 0, xj = valid ? (int)r.w : 0;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const int tc = __shfl_up_sync(0xffffffffu, xc, d), tj = __shfl_up_sync(0xffffffffu, xj, d);
            if (lane >= d) {
                xc += tc;
                xj += tj;
            }
        }
        const int cc = cum_c + xc, cj = cum_j + xj;  // inclusive running sums at i
        const unsigned ends = __ballot_sync(0xffffffffu, is_end);
        const unsigned below = ends & lt;
        const int src = below ? 31 - __clz(below) : lane;  // previous run end in this window
        const int pcv = __shfl_sync(0xffffffffu, cc, src), pjv = __shfl_sync(0xffffffffu, cj, src);
        const int bc = below ? pcv : end_c, bj = below ? pjv : end_j;
        const bool ec = is_end && cc != bc, eo = is_end && cj != bj;
        const unsigned mc = __ballot_sync(0xffffffffu, ec), mo = __ballot_sync(0xffffffffu, eo);
        if (EMIT) {
            const double h = key_height(k);
            if (ec) {
                const long long pos = pc + __popc(mc & lt);
                if (a.do_ect) {
                    reinterpret_cast<double *>(a.ect.h)[pos] = h;
                    reinterpret_cast<int64_t *>(a.ect.v)[pos] = cc;
                }
                if (a.do_cls) {
                    if (!a.cls_alias) reinterpret_cast<double *>(a.cls.h)[pos] = h;
                    reinterpret_cast<int64_t *>(a.cls.v)[pos] = (int64_t)bj + (cc - bc);
                }
            }
            if (eo && a.do_ord) {
                const long long pos = po + __popc(mo & lt);
                reinterpret_cast<double *>(a.ord.h)[pos] = h;
                reinterpret_cast<int64_t *>(a.ord.v)[pos] = cj;
            }
        }
        pc += __popc(mc);
        po += __popc(mo);
        nc += __popc(mc);
        no += __popc(mo);
        cum_c = __shfl_sync(0xffffffffu, cc, 31);
        cum_j = __shfl_sync(0xffffffffu, cj, 31);
        if (ends) {
            const int le = 31 - __clz(ends);
            end_c = __shfl_sync(0xffffffffu, cc, le);
            end_j = __shfl_sync(0xffffffffu, cj, le);
        }
    }
    sc = cum_c - ic;
    sj = cum_j - ij;
}

constexpr int kPieceWarps = kThreads / 32;

template <bool EMIT>
__global__ void __launch_bounds__(kThreads) k5b_piece(K5Args a, K5Big g) {
    extern __shared__ uint4 k5b_buf[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint4 *buf = k5b_buf + warp * kK5PieceMax;
    for (long long p = (long long)blockIdx.x * kPieceWarps + warp; p < g.npieces;
         p += (long long)gridDim.x * kPieceWarps) {
        const int len = g.p_len[p];
        const long long st = g.p_start[p];
        const uint4 *src = g.scr + st;
        int nc, no, sc, sj;
        if (!EMIT) {
            if (len > 1 && len <= kK5PieceMax) {
                int np = 2;
                while (np < len) np <<= 1;
                for (int i = lane; i < np; i += 32) buf[i] = i < len ? src[i] : make_uint4(~0u, ~0u, 0u, 0u);
                __syncwarp();
                for (int k = 2; k <= np; k <<= 1)
                    for (int j = k >> 1; j > 0; j >>= 1) {
                        for (int u = lane; u < (np >> 1); u += 32) {
                            const int i = ((u & ~(j - 1)) << 1) | (u & (j - 1)), q = i | j;
                            const bool up = (i & k) == 0;
                            const uint4 x = buf[i], y = buf[q];
                            const unsigned long long kx = rec_key(x), ky = rec_key(y);
                            if (up ? (kx > ky) : (kx < ky)) {
                                buf[i] = y;
                                buf[q] = x;
                            }
                        }
                        __syncwarp();
                    }
                for (int i = lane; i < len; i += 32) g.scr[st + i] = buf[i];  // sorted, for the emit pass
                src = buf;
            }
            rle_piece<false>(a, src, len, 0, 0, 0, 0, nc, no, sc, sj);
            if (lane == 0) {
                g.p_nc[p] = nc;
                g.p_no[p] = no;
                g.p_sc[p] = sc;
                g.p_sj[p] = sj;
            }
        } else {
            const long long s = g.seg[g.p_seg[p]];
            const long long pc = (a.do_ect ? a.ect.off[s] : a.do_cls ? a.cls.off[s] : 0) + g.p_offc[p];
            const long long po = (a.do_ord ? a.ord.off[s] : 0) + g.p_offo[p];
            rle_piece<true>(a, src, len, g.p_ic[p], g.p_ij[p], pc, po, nc, no, sc, sj);
        }
        __syncwarp();
    }
}

__global__ void __launch_bounds__(kBigThreads) k5b_segscan(K5Args a, K5Big g) {
    const long long i = blockIdx.x;
    const long long s = g.seg[i], pb = g.pbase[i];
    const int nb = g.nb[i];
    const int per = (nb + blockDim.x - 1) / blockDim.x;
    const int k0 = min(nb, (int)threadIdx.x * per), k1 = min(nb, k0 + per);
    int v[4] = {0, 0, 0, 0}, tot[4];
    for (int k = k0; k < k1; ++k) {
        v[0] += g.p_nc[pb + k];
        v[1] += g.p_no[pb + k];
        v[2] += g.p_sc[pb + k];
        v[3] += g.p_sj[pb + k];
    }
    block_excl_scan<4>(v, tot);
    for (int k = k0; k < k1; ++k) {
        const long long p = pb + k;
        g.p_offc[p] = v[0];
        g.p_offo[p] = v[1];
        g.p_ic[p] = v[2];
        g.p_ij[p] = v[3];
        v[0] += g.p_nc[p];
        v[1] += g.p_no[p];
        v[2] += g.p_sc[p];
        v[3] += g.p_sj[p];
    }
    if (threadIdx.x == 0) {
        a.cnt_c[s] = tot[0];
        a.cnt_o[s] = tot[1];
    }
}

template <typename RecT>
cudaError_t launch_bucket(const K5Args &a, const K5Big &g, int nb_max, cudaStream_t s) {
    auto k = k5b_bucket<RecT>;
    const size_t smem = sizeof(unsigned) * (size_t)std::max(nb_max, 1);
    cudaError_t e = prepare_kernel((const void *)k, kBigThreads, smem, nullptr);
    if (e != cudaSuccess) return e;
    k<<<(unsigned)g.nseg, kBigThreads, smem, s>>>(a, g);
    count_launch();
    return cudaGetLastError();
}

}  // namespace

size_t k5_smem(int npow2) { return (size_t)npow2 * 16; }

cudaError_t launch_k5(const K5Args &a, int phase, cudaStream_t s, int num_sms) {
    return a.wide ? launch_r<Rec32>(a, phase, s, num_sms) : launch_r<Rec16>(a, phase, s, num_sms);
}

cudaError_t launch_k5_scan(const K5Args &a, cudaStream_t s) {
    return launch_csr_scan(a.scan, a.cnt_c, a.cnt_o, a.batch * a.D, s);
}

cudaError_t launch_k5b_prepare(const K5Args &a, const K5Big &g, int nb_max, cudaStream_t s, int num_sms) {
    if (g.nseg == 0) return cudaSuccess;
    cudaError_t e = cudaMemsetAsync(g.over, 0, 2 * sizeof(unsigned), s);
    if (e == cudaSuccess) e = a.wide ? launch_bucket<Rec32>(a, g, nb_max, s) : launch_bucket<Rec16>(a, g, nb_max, s);
    if (e != cudaSuccess) return e;
    {
        const size_t smem = sizeof(uint4) * kSortTile;
        e = prepare_kernel((const void *)k5b_sort, kBigThreads, smem, nullptr);
        if (e != cudaSuccess) return e;
        k5b_sort<<<(unsigned)num_sms, kBigThreads, smem, s>>>(g);
    }
    {
        const size_t smem = sizeof(uint4) * kK5PieceMax * kPieceWarps;
        int occ = 0;
        e = prepare_kernel((const void *)k5b_piece<false>, kThreads, smem, &occ);
        if (e != cudaSuccess) return e;
        const long long grid =
            std::min<long long>((g.npieces + kPieceWarps - 1) / kPieceWarps, (long long)std::max(occ, 1) * num_sms);
        k5b_piece<false><<<(unsigned)std::max<long long>(grid, 1), kThreads, smem, s>>>(a, g);
    }
    k5b_segscan<<<(unsigned)g.nseg, kBigThreads, 0, s>>>(a, g);
    count_launch(3);
    return cudaGetLastError();
}

cudaError_t launch_k5b_emit(const K5Args &a, const K5Big &g, cudaStream_t s, int num_sms) {
    if (g.nseg == 0) return cudaSuccess;
    int occ = 0;
    cudaError_t e = prepare_kernel((const void *)k5b_piece<true>, kThreads, 0, &occ);
    if (e != cudaSuccess) return e;
    const long long grid =
        std::min<long long>((g.npieces + kPieceWarps - 1) / kPieceWarps, (long long)std::max(occ, 1) * num_sms);
    k5b_piece<true><<<(unsigned)std::max<long long>(grid, 1), kThreads, 0, s>>>(a, g);
    count_launch();
    return cudaGetLastError();
}

}  // namespace eucalc
