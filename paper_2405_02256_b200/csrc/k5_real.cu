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
cudaError_t launch_r(const K5Args &a, cudaStream_t s, int num_sms) {
    const size_t per_warp = (size_t)a.npow2 * 16;
    const int wpb = (int)std::max<size_t>(1, std::min<size_t>(kThreads / 32, (size_t)(64 * 1024) / per_warp));
    const size_t smem = per_warp * wpb;
    auto kc = k5_real<RecT, int64_t, false>;
    auto ke = k5_real<RecT, int64_t, true>;
    int occ = 0;
    cudaError_t e = prepare_kernel((const void *)kc, wpb * 32, smem, &occ);
    if (e == cudaSuccess) e = prepare_kernel((const void *)ke, wpb * 32, smem, nullptr);
    if (e != cudaSuccess) return e;
    const long long S = a.batch * a.D;
    const long long grid = std::min<long long>((S + wpb - 1) / wpb, (long long)std::max(occ, 1) * num_sms);
    kc<<<(unsigned)grid, wpb * 32, smem, s>>>(a, wpb);
    e = launch_csr_scan(a.scan, a.cnt_c, a.cnt_o, S, s);
    if (e != cudaSuccess) return e;
    ke<<<(unsigned)grid, wpb * 32, smem, s>>>(a, wpb);
    count_launch(2);
    return cudaGetLastError();
}

}  // namespace

size_t k5_smem(int npow2) { return (size_t)npow2 * 16; }

cudaError_t launch_k5(const K5Args &a, cudaStream_t s, int num_sms) {
    return a.wide ? launch_r<Rec32>(a, s, num_sms) : launch_r<Rec16>(a, s, num_sms);
}

}  // namespace eucalc
