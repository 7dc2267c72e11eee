// K4 — evaluation and vectorisation of the exact representations (NEXT row f1;
// P:135-137 evaluation by binary search, P:339-341 vectorisation).
//
//   ECT(xi, t)   = E[i], i the last breakpoint with height <= t (0 if none)
//   Radon(xi, t) = E_c[j] if t is a classical height T_c[j], else E'[i],
//                  i the last ordinary breakpoint strictly below t (E7)
//
// t is a double in the paper's normalised units. Breakpoints are
// integer lattice heights H with t(H) = (2H - L*csum) / (2L) (E10), so every
// comparison is decided exactly in integers: F = floor(2L t) is formed from the
// rounded product p = 2L*t and its exact error e = fma(2L, t, -p) (an
// error-free transformation), and
//   t(H) <= t  <=>  2H - L*csum <= F         (H <= Hle)
//   t(H) <  t  <=>  the same with F - 1 when 2L t is an integer (H <= Hlt)
//   t(H) == t  <=>  2L t is an integer and F + L*csum = 2H.
// Vectorisation generates t_i = a + (i*(b-a))/(N-1) with round-to-nearest
// intrinsics (no contraction into an FMA), the exact double sequence the oracle
// uses (E20).
//
// One thread per (segment, query): a binary search over the segment's
// breakpoints (read through L1; a segment's heights are contiguous). Bound:
// the output write plus the log-depth reads.
#include <algorithm>
#include <cmath>

#include "eucalc_internal.cuh"

namespace eucalc {
namespace {

constexpr int kThreads = 256;
constexpr long long kBig = 1ll << 62;

struct Threshold {
    long long le;     // largest lattice height H with t(H) <= t
    long long lt;     // largest lattice height H with t(H) <  t
    long long exact;  // H with t(H) == t, or kBig if t is not a lattice height
    bool nan;
};

__device__ __forceinline__ long long floor_div2(long long x) { return x >= 0 ? x / 2 : -((1 - x) / 2); }

__device__ __forceinline__ Threshold threshold(double t, long long L2, long long Lc) {
    Threshold r;
    r.nan = isnan(t);
    r.exact = kBig;
    const double p = __dmul_rn((double)L2, t);
    if (r.nan) {
        r.le = r.lt = -kBig;
        return r;
    }
    if (p >= 4503599627370496.0) {  // 2^52: beyond every height (|H| < 2^31)
        r.le = r.lt = kBig;
        return r;
    }
    if (p <= -4503599627370496.0) {
        r.le = r.lt = -kBig;
        return r;
    }
    const double e = fma((double)L2, t, -p);  // 2L t = p + e exactly
    const double f = floor(p);
    long long F = (long long)f;
    const bool integral = f == p;
    if (integral && e < 0.0) F -= 1;
    const bool exact = integral && e == 0.0;
    const long long X = F + Lc;
    r.le = floor_div2(X);
    r.lt = exact ? floor_div2(X - 1) : r.le;
    if (exact && (X & 1) == 0) r.exact = X / 2;
    return r;
}

// number of entries of h[0..n) that are <= x (h ascending)
template <typename T>
__device__ __forceinline__ long long upper_bound(const T *h, long long n, long long x) {
    long long lo = 0, hi = n;
    while (lo < hi) {
        const long long mid = (lo + hi) >> 1;
        if ((long long)h[mid] <= x) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

template <typename InT, typename OutT>
__global__ void __launch_bounds__(kThreads) k4_eval(K4Args a) {
    const long long S = a.batch * a.D;
    const long long total = S * a.nq;
    const InT *rh = (const InT *)a.rep_h, *rv = (const InT *)a.rep_v;
    const InT *ch = (const InT *)a.cls_h, *cv = (const InT *)a.cls_v;
    OutT *out = (OutT *)a.out;
    // one thread per (segment, query): consecutive threads take consecutive
    // queries of a segment (coalesced output; the segment's breakpoints are
    // shared through L1), so a few segments with many points (vectorisation of
    // one large image) spread over the whole GPU as well
    for (long long item = (long long)blockIdx.x * kThreads + threadIdx.x; item < total;
         item += (long long)gridDim.x * kThreads) {
        const long long s = item / a.nq, q = item - s * a.nq;
        const long long d = s % a.D;
        const long long L2 = 2 * a.L, Lc = a.L * (long long)a.csum[d];
        const long long r0 = a.rep_off[s], rn = a.rep_off[s + 1] - r0;
        double t;
        if (a.t) {
            t = a.t[q];
        } else if (a.nq == 1) {
            t = a.ta;
        } else {
            t = __dadd_rn(a.ta, __ddiv_rn(__dmul_rn((double)q, __dsub_rn(a.tb, a.ta)), (double)(a.nq - 1)));
        }
        const Threshold th = threshold(t, L2, Lc);
        long long v = 0;
        if (!th.nan) {
            if (a.kind == EUCALC_EVAL_ECT) {
                const long long i = upper_bound(rh + r0, rn, th.le);
                v = i ? (long long)rv[r0 + i - 1] : 0;
            } else {
                const long long c0 = a.cls_off[s], cn = a.cls_off[s + 1] - c0;
                bool hit = false;
                if (th.exact != kBig && cn) {
                    const long long j = upper_bound(ch + c0, cn, th.exact);
                    if (j && (long long)ch[c0 + j - 1] == th.exact) {
                        v = (long long)cv[c0 + j - 1];
                        hit = true;
                    }
                }
                if (!hit) {
                    const long long i = upper_bound(rh + r0, rn, th.lt);
                    v = i ? (long long)rv[r0 + i - 1] : 0;
                }
            }
        }
        out[item] = (OutT)v;
    }
}

template <typename InT>
cudaError_t launch_in(const K4Args &a, cudaStream_t s, int num_sms) {
    const long long total = a.batch * a.D * a.nq;
    const long long blocks = std::min<long long>((total + kThreads - 1) / kThreads, 16ll * num_sms);
    if (a.out_eb == 4) k4_eval<InT, int32_t><<<(unsigned)blocks, kThreads, 0, s>>>(a);
    else k4_eval<InT, int64_t><<<(unsigned)blocks, kThreads, 0, s>>>(a);
    count_launch();
    return cudaGetLastError();
}

}  // namespace

cudaError_t launch_k4(const K4Args &a, cudaStream_t s, int num_sms) {
    if (a.batch * a.D == 0 || a.nq == 0) return cudaSuccess;
    switch (a.in_eb) {
    case 2: return launch_in<int16_t>(a, s, num_sms);
    case 4: return launch_in<int32_t>(a, s, num_sms);
    default: return launch_in<int64_t>(a, s, num_sms);
    }
}

}  // namespace eucalc
