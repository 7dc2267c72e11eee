// K3 — hybrid transform.
//
// HT(xi) = int kappa(t) Radon(xi,t) dt = - sum_{ordinary x} J(eps,x) kbar(t(x))
// (Lemma 2, ordinary sign corrected E1; "we sum, over all
// ordinary critical points, the evaluation of the kernel kbar on the dot
// products"), t(x) the paper's normalised height:
//   t = (2H - L*csum) / (2L),  H = sum_i xs_i p_i an exact integer (E10, E11).
// The additive constant of kbar cancels because sum J = 0.
//
// Work decomposition: directions are grouped by orthant on the host (Lemma 3,
// same sign vector -> same critical list) into tiles of <= 512; a CTA
// owns (image, tile, chunk of kChunk records) with one direction per thread in
// registers and the chunk staged in shared memory (broadcast reads). Per term
// (k3_f64, the per-term "direct" algorithm): the exact integer height, kbar
// (erf / sinpi with exact integer period reduction / cos / exp) and one FMA,
// all in fp64 for both output precisions: an fp32 kbar rounds every term by up
// to an ulp, and on ill-conditioned directions (sum |J kbar| / |HT| up to 1e7
// in config 5) that alone exceeds the fp32 tolerance (measured 7e-4 absolute).
// Chunk partials are combined in a fixed order by a second kernel, so results
// are bit-identical run to run.
#include <cmath>
#include <type_traits>

#include "eucalc_internal.cuh"

namespace eucalc {
namespace {

constexpr int kThreads = 512;  // max block: one direction per thread, tiles of <= 512
constexpr int kChunk = 4096;
constexpr int kStage = 1024;

template <typename RecT>
__device__ __forceinline__ void rec_coords(const RecT &r, const K3Args &a, int &p0, int &p1, int &p2) {
    p0 = (int)((r.c >> a.sh[0]) & a.msk[0]);
    p1 = (int)((r.c >> a.sh[1]) & a.msk[1]);
    p2 = (a.ndim == 3) ? (int)((r.c >> a.sh[2]) & a.msk[2]) : 0;
}

template <typename RecT>
__global__ void __launch_bounds__(kThreads) k3_f64(K3Args a) {
    __shared__ int4 sm[kStage];
    const int c = blockIdx.x, tile = blockIdx.y;
    const long long b = blockIdx.z;
    const int tlen = a.tile_len[tile];
    const int myd = threadIdx.x < tlen ? a.order[a.tile_start[tile] + threadIdx.x]
                                       : a.order[a.tile_start[tile]];
    const DirInfo di = a.dirs[myd];
    const DirInfo di0 = a.dirs[a.order[a.tile_start[tile]]];
    const int n = a.count[b * a.Q + di0.q];
    const RecT *list = reinterpret_cast<const RecT *>(a.rec) + (b * a.Q + di0.q) * a.vcap;
    const int beg = c * a.chunk, end = min(n, beg + a.chunk);
    const int x0 = di.xs[0], x1 = di.xs[1], x2 = (a.ndim == 3) ? di.xs[2] : 0;
    const double L = (double)a.L;
    const double cs = (double)a.csum[myd];
    double c1 = 0, c0 = 0, per = 0, inv_per = 0, inv_half = 0;
    bool int_period = false;
    if (a.kernel == EUCALC_K_GAUSS) {
        const double k = 1.0 / (a.param * sqrt(2.0));
        c1 = k / L;
        c0 = -0.5 * cs * k;
    } else if (a.kernel == EUCALC_K_COS) {
        const double lp = L * a.param;
        int_period = (a.param == rint(a.param)) && lp < 1.0e15;
        per = 2.0 * lp;
        inv_per = 1.0 / per;
        inv_half = 1.0 / lp;
        c0 = -L * cs;
        c1 = 2.0 * M_PI / a.param / (2.0 * L);
    } else {
        c1 = 1.0 / L;
        c0 = -0.5 * cs;
    }
    double acc0 = 0.0, acc1 = 0.0;
    const int sw = di.swap;
    for (int s0 = beg; s0 < end; s0 += kStage) {
        const int cnt = min(kStage, end - s0);
        __syncthreads();
        for (int i = threadIdx.x; i < cnt; i += blockDim.x) {
            const RecT r = list[s0 + i];
            int p0, p1, p2;
            rec_coords(r, a, p0, p1, p2);
            sm[i] = make_int4(p0, p1, p2, sw ? (r.b - r.a) : (r.a - r.b));
        }
        __syncthreads();
        if (threadIdx.x < tlen) {
#pragma unroll 2
            for (int i = 0; i < cnt; ++i) {
                const int4 r = sm[i];
                const double h = (double)(r.x * x0 + r.y * x1 + r.z * x2);  // exact integer
                double kb;
                if (a.kernel == EUCALC_K_GAUSS) {
                    kb = erf(fma(h, c1, c0));
                } else if (a.kernel == EUCALC_K_COS) {
                    const double u = fma(2.0, h, c0);
                    if (int_period) {
                        const double q = rint(u * inv_per);
                        kb = sinpi(fma(-q, per, u) * inv_half);
                    } else {
                        kb = sin(u * c1);
                    }
                } else if (a.kernel == EUCALC_K_SIN) {
                    kb = cos(fma(h, c1, c0));
                } else {
                    kb = exp(fma(h, c1, c0));
                }
                if (i & 1) acc1 = fma((double)r.w, kb, acc1);
                else acc0 = fma((double)r.w, kb, acc0);
            }
        }
    }
    if (threadIdx.x < tlen) a.partial[(b * a.nchunks + c) * a.D + myd] = acc0 + acc1;
}

// ---------------------------------------------------------------------------
// Tabulated kbar (the default path). t depends on the record only through the
// integer u = 2H - L*csum (E10), so kbar(t(u)) is evaluated ONCE per u over the
// range the directions span, in fp64 (the same formulas and the same exact
// integer period reduction as above), and every term becomes a table lookup:
//   idx = H + off_d  (one dp2a/dp4a on the packed coordinates; off_d folds in
//                     -L*csum_d and the table origin, u halved: a tile's
//                     directions share the parity of L*csum, hence of u),
//   acc += J * tab[idx].
// The half table of the tile's parity sits in shared memory; per term the work
// is an LDS broadcast of the record, a DP4A, an LDS gather and the accumulation
// — precision-independent kbar cost, no SFU. Table element and accumulation per
// mode (K3Mode):
//   kF64  : fp64 kbar, DFMA (fp64 output);
//   kFix32: the bounded kernels' f = erf / sinpi / cos in [-1, 1] as 32-bit fixed
//           point q = rint(f 2^30) (|error| <= 2^-31), J * q accumulated EXACTLY in
//           int64 (IMAD.WIDE; |J q| < 2^47, <= 8192 terms per CTA): the fp32
//           output path. The table's rounding errors are independent per lattice
//           height, so the HT error is ~2^-31 sqrt(sum_h H_J(h)^2) — 1e-5 on the
//           worst-conditioned config-5 directions, where fp32 kbar values
//           (rounded by up to 2^-24) reach 1e-4 (E23);
//   kF32  : fp32 kbar with Kahan-compensated fp32 accumulation (EXP, whose kbar is
//           unbounded, and int32-weight records).
constexpr int kChunkT = 8192;
constexpr int kFixBits = 30;
enum K3Mode { kF32 = 0, kF64 = 1, kFix32 = 2 };

// split = 1 (fused HT in K2): t64 holds the even-offset entries (u - U0 even)
// first, then the odd ones, so one direction's entries (fixed parity of u) are
// contiguous in its heights; t32 (natural order) may be NULL and holds float
// values, or int32 fixed-point values when fix32 = 1.
__global__ void k3_table(int kernel, double param, long long L, long long U0, long long U, double *t64, float *t32,
                         int split = 0, int fix32 = 0) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= U) return;
    const long long u = U0 + i;
    double f;
    if (kernel == EUCALC_K_GAUSS) {
        f = erf((double)u * (1.0 / (param * sqrt(2.0))) / (2.0 * (double)L));
    } else if (kernel == EUCALC_K_COS) {
        const double lp = (double)L * param;
        if (param == rint(param) && lp < 1.0e15) {
            const long long per = 2 * (long long)lp;  // period of u
            long long r = u % per;
            if (r < 0) r += per;
            f = sinpi((double)r / lp);
        } else {
            f = sin((double)u * M_PI / lp);
        }
    } else if (kernel == EUCALC_K_SIN) {
        f = cos((double)u / (2.0 * (double)L));
    } else {
        f = exp((double)u / (2.0 * (double)L));
    }
    t64[split ? ((i & 1) ? ((U + 1) >> 1) + (i >> 1) : (i >> 1)) : i] = f;
    if (t32) {
        if (fix32) reinterpret_cast<int *>(t32)[i] = (int)rint(f * (double)(1 << kFixBits));
        else t32[i] = (float)f;
    }
}

template <int DP>
__device__ __forceinline__ int table_index(uint32_t c, int xs8, int off) {
    int r;
    if (DP == 2) asm("dp2a.lo.u32.s32 %0, %1, %2, %3;" : "=r"(r) : "r"(c), "r"(xs8), "r"(off));
    else asm("dp4a.u32.s32 %0, %1, %2, %3;" : "=r"(r) : "r"(c), "r"(xs8), "r"(off));
    return r;
}

template <typename RecT, int MODE, int DP>
__global__ void __launch_bounds__(kThreads) k3t(K3Args a) {
    constexpr bool F64 = MODE == kF64, FIX = MODE == kFix32;
    using T = typename std::conditional<F64, double, typename std::conditional<FIX, int, float>::type>::type;
    using S = typename std::conditional<F64, int4, int2>::type;  // staged record: c, J (int / float bits / double)
    using Acc = typename std::conditional<F64, double, typename std::conditional<FIX, long long, float>::type>::type;
    constexpr int PER = F64 ? 2 : 4;                             // records staged per thread per chunk
    extern __shared__ __align__(16) unsigned char k3t_smem[];
    S *sbuf = reinterpret_cast<S *>(k3t_smem);  // two staging buffers of PER * blockDim records
    const int stage_n = PER * blockDim.x;
    T *tab = reinterpret_cast<T *>(sbuf + 2 * PER * kThreads);
    const int c = blockIdx.x, tile = blockIdx.y;
    const long long b = blockIdx.z;
    const int tlen = a.tile_len[tile];
    const int d0 = a.order[a.tile_start[tile]];
    const int myd = threadIdx.x < tlen ? a.order[a.tile_start[tile] + threadIdx.x] : d0;
    const DirInfo di = a.dirs[myd];
    const DirInfo di0 = a.dirs[d0];
    const int n = a.count[b * a.Q + di0.q];
    const int beg = c * a.chunk, end = min(n, beg + a.chunk);
    // the tile's half table: u = start + 2 j, u == L*csum (mod 2)
    const int par = (int)((a.L * (long long)a.csum[d0]) & 1);
    const long long start = a.U0 + (((a.U0 & 1) != par) ? 1 : 0);
    const int half = (int)((a.U0 + a.U - 1 - start) / 2 + 1);
    const T *gtab = F64 ? reinterpret_cast<const T *>(a.tab64) : reinterpret_cast<const T *>(a.tab32);
    for (int j = threadIdx.x; j < half; j += blockDim.x) tab[j] = gtab[start - a.U0 + 2 * (long long)j];
    // idx = (u - start) / 2 = H + off, off = (-L*csum - start) / 2 (exact: same parity)
    const int off = (int)((-a.L * (long long)a.csum[myd] - start) / 2);
    // H = sum xs_k p_k = dp(c, xs8): records carry the vertex coordinates; the
    // pair's representative orthant is this direction's orthant up to the
    // antipodal swap (J -> -J, handled at staging)
    const int sw = di0.swap;
    const RecT *list = reinterpret_cast<const RecT *>(a.rec) + (b * a.Q + di0.q) * a.vcap;
    // staging, double-buffered: the next chunk's records are loaded into
    // registers before the current chunk is consumed, and stored after it
    RecT pre[PER];
    auto load_chunk = [&](int s0) {
#pragma unroll
        for (int k = 0; k < PER; ++k) {
            const int i = s0 + k * blockDim.x + threadIdx.x;
            if (i < end) pre[k] = list[i];
        }
    };
    auto store_chunk = [&](S *dst, int s0) {
#pragma unroll
        for (int k = 0; k < PER; ++k) {
            const int li = k * blockDim.x + threadIdx.x;
            if (s0 + li < end) {
                const int j = sw ? (pre[k].b - pre[k].a) : (pre[k].a - pre[k].b);
                if constexpr (F64) {
                    const double jd = (double)j;
                    dst[li] = make_int4((int)pre[k].c, 0, __double2loint(jd), __double2hiint(jd));
                } else if constexpr (FIX) {
                    dst[li] = make_int2((int)pre[k].c, j);
                } else {
                    dst[li] = make_int2((int)pre[k].c, __float_as_int((float)j));
                }
            }
        }
    };
    Acc acc0 = 0, acc1 = 0;
    float cmp0 = 0.f, cmp1 = 0.f;  // Kahan compensation (kF32)
    auto add = [&](Acc &acc, float &cmp, const S &r, T k) {
        if constexpr (F64) {
            acc = fma(__hiloint2double(r.w, r.z), k, acc);
        } else if constexpr (FIX) {
            acc += (long long)r.y * (long long)k;  // exact (IMAD.WIDE)
        } else {
            // Kahan-compensated fp32 (J * kbar formed inside the FMA)
            const float y = fmaf(__int_as_float(r.y), k, -cmp), t = acc + y;
            cmp = (t - acc) - y;
            acc = t;
        }
    };
    if (beg < end) {
        load_chunk(beg);
        store_chunk(sbuf, beg);
    }
    __syncthreads();
    int cur = 0;
    for (int s0 = beg; s0 < end; s0 += stage_n) {
        const int cnt = min(stage_n, end - s0);
        const int nxt = s0 + stage_n;
        if (nxt < end) load_chunk(nxt);  // in flight while this chunk is consumed
        const S *srec = sbuf + cur * PER * kThreads;
        if (threadIdx.x < tlen) {
            // four independent record chains per iteration (LDS -> IDP -> LDS -> accumulate)
            int i = 0;
            for (; i + 3 < cnt; i += 4) {
                S r[4];
                T k[4];
                if constexpr (F64) {
#pragma unroll
                    for (int u = 0; u < 4; ++u) r[u] = srec[i + u];
                } else {
                    // two records per 16-byte broadcast load
                    const int4 p0 = *reinterpret_cast<const int4 *>(srec + i);
                    const int4 p1 = *reinterpret_cast<const int4 *>(srec + i + 2);
                    r[0] = make_int2(p0.x, p0.y);
                    r[1] = make_int2(p0.z, p0.w);
                    r[2] = make_int2(p1.x, p1.y);
                    r[3] = make_int2(p1.z, p1.w);
                }
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    EU_DCHECK((unsigned)table_index<DP>((uint32_t)r[u].x, di.xs8, off) < (unsigned)half);
                    k[u] = tab[table_index<DP>((uint32_t)r[u].x, di.xs8, off)];
                }
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    if (u & 1) add(acc1, cmp1, r[u], k[u]);
                    else add(acc0, cmp0, r[u], k[u]);
                }
            }
            for (; i < cnt; ++i) {
                const S r0 = srec[i];
                EU_DCHECK((unsigned)table_index<DP>((uint32_t)r0.x, di.xs8, off) < (unsigned)half);
                add(acc0, cmp0, r0, tab[table_index<DP>((uint32_t)r0.x, di.xs8, off)]);
            }
        }
        if (nxt < end) store_chunk(sbuf + (cur ^ 1) * PER * kThreads, nxt);
        __syncthreads();
        cur ^= 1;
    }
    if (threadIdx.x < tlen) {
        double tot;
        if constexpr (F64) tot = acc0 + acc1;
        else if constexpr (FIX) tot = (double)(acc0 + acc1) * (1.0 / (double)(1 << kFixBits));
        else tot = ((double)acc0 - (double)cmp0) + ((double)acc1 - (double)cmp1);
        a.partial[(b * a.nchunks + c) * a.D + myd] = tot;
    }
}

// Fixed-order combine of the chunk partials; applies -scale of kbar.
__global__ void k3_combine(const K3Args a, double scale) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= a.batch * a.D) return;
    const long long b = i / a.D, d = i % a.D;
    double s = 0.0;
    for (int c = 0; c < a.nchunks; ++c) s += a.partial[(b * a.nchunks + c) * a.D + d];
    const double v = scale * s;
    if (a.precision == EUCALC_F32) reinterpret_cast<float *>(a.out)[i] = (float)v;
    else reinterpret_cast<double *>(a.out)[i] = v;
}

}  // namespace

int k3_chunk(bool table) { return table ? kChunkT : kChunk; }

// Table mode of a K3 call: fp64 output -> kF64; fp32 output -> kFix32 for the
// bounded kernels over 16-bit-weight records, else kF32.
int k3_mode(int kernel, int precision, bool wide) {
    if (precision == EUCALC_F64) return kF64;
    return (kernel != EUCALC_K_EXP && !wide) ? kFix32 : kF32;
}

size_t k3_table_smem(int mode, long long U) {
    const long long half = (U + 1) / 2 + 1;
    // two staging buffers of PER * kThreads records (PER = 2 in fp64, 4 otherwise)
    return (mode == kF64 ? sizeof(int4) * 2 : sizeof(int2) * 4) * 2 * kThreads + (mode == kF64 ? 8 : 4) * half;
}

cudaError_t launch_k3_table(const K3Args &a, cudaStream_t s) {
    // kbar table over u in [U0, U0 + U)
    k3_table<<<(unsigned)((a.U + 255) / 256), 256, 0, s>>>(a.kernel, a.param, a.L, a.U0, a.U, a.tab64, a.tab32, 0,
                                                           k3_mode(a.kernel, a.precision, a.wide) == kFix32);
    count_launch();
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    return cudaSuccess;
}

cudaError_t launch_k3_table_only(int kernel, double param, int64_t L, int64_t U0, int64_t U, double *t64, float *t32,
                                 cudaStream_t s) {
    k3_table<<<(unsigned)((U + 255) / 256), 256, 0, s>>>(kernel, param, L, U0, U, t64, t32, 1);
    count_launch();
    return cudaGetLastError();
}

double k3_scale(int kernel, double param) {
    // HT = -sum J kbar; kbar = scale_k * f  (f is what the table holds)
    switch (kernel) {
    case EUCALC_K_GAUSS: return -param * sqrt(M_PI / 2.0);
    case EUCALC_K_COS: return -param / (2.0 * M_PI);
    case EUCALC_K_SIN: return 1.0;  // kbar = -cos
    default: return -1.0;           // kbar = exp
    }
}

cudaError_t launch_k3(const K3Args &a, cudaStream_t s) {
    dim3 grid((unsigned)a.nchunks, (unsigned)a.ntiles, (unsigned)a.batch);
    if (a.use_table) {
        cudaError_t e = launch_k3_table(a, s);
        if (e != cudaSuccess) return e;
        const int mode = k3_mode(a.kernel, a.precision, a.wide);
        const size_t smem = k3_table_smem(mode, a.U);
        void (*k)(K3Args) = nullptr;
        if (a.wide) {
            if (mode == kF64) k = a.dp == 2 ? k3t<Rec32, kF64, 2> : k3t<Rec32, kF64, 3>;
            else k = a.dp == 2 ? k3t<Rec32, kF32, 2> : k3t<Rec32, kF32, 3>;
        } else {
            if (mode == kF64) k = a.dp == 2 ? k3t<Rec16, kF64, 2> : k3t<Rec16, kF64, 3>;
            else if (mode == kFix32) k = a.dp == 2 ? k3t<Rec16, kFix32, 2> : k3t<Rec16, kFix32, 3>;
            else k = a.dp == 2 ? k3t<Rec16, kF32, 2> : k3t<Rec16, kF32, 3>;
        }
        e = prepare_kernel((const void *)k, a.threads, smem, nullptr);
        if (e != cudaSuccess) return e;
        k<<<grid, a.threads, smem, s>>>(a);
    } else {
        // per-term kbar in fp64 for both output precisions (see k3_f64)
        if (a.wide) k3_f64<Rec32><<<grid, a.threads, 0, s>>>(a);
        else k3_f64<Rec16><<<grid, a.threads, 0, s>>>(a);
    }
    count_launch();
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    const double scale = k3_scale(a.kernel, a.param);
    const long long tot = a.batch * a.D;
    k3_combine<<<(unsigned)((tot + 255) / 256), 256, 0, s>>>(a, scale);
    count_launch();
    return cudaGetLastError();
}

}  // namespace eucalc
