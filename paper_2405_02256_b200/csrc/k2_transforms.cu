// K2 — exact ECT and Radon representations (SURVEY 8(a) A3 heights, A4 sort +
// run-length merge, A5 scan + emit).
//
// Lemma 2 (ordinary sign corrected, E1), for direction xi in orthant eps:
//   ECT(xi,.)   = sum_{x} Delta^-(eps,x) 1_[h(x), +inf)
//   Radon(xi,.) = sum_{x} Delta^-(eps,x) 1_{h(x)} + sum_{x} J(eps,x) 1_(h(x), +inf)
// The paper sorts the dots and takes cumulative sums, merging equal dots
// (P:126-128). Heights here are integers in a known range [hlo, hlo+R) (E10),
// so the final pass of a radix sort degenerates to a weighted histogram over
// the R lattice heights: bin h accumulates (sum Delta^-, sum J) of the records
// at height h — the run-length merge, with no permutation materialised. One
// 64-bit shared-memory atomic per record adds both sums at once
// (packed = J * 2^32 + Delta^-; exact while |sums| < 2^31, checked on the host).
// A scan over the bins then emits, in ascending height order,
//   ECT       : (h, E)   at bins with sum Delta^- != 0           (E8: zero-net dropped)
//   ordinary  : (h, E')  at bins with sum J != 0,  E' = Radon(h+)
//   classical : (h, E_c) at bins with sum Delta^- != 0, E_c = Radon(h-) + sum Delta^-
// (T_c = T by Lemma 6). Output offsets of segment s = image*D + dir come
// from a decoupled look-back in ticket order, so the CSR is written in one
// pass and is bit-identical run to run.
//
// Two regimes (SURVEY 7 hard part 2):
//   warp kernel : one warp per segment, whole histogram (R <= a few thousand
//                 bins) in a warp-private smem slab; lists of the CTA's image
//                 read through L1 (configs 1-2: ~10^3 tiny problems).
//   block kernel: one CTA per segment, heights processed in windows of up to
//                 kWinBins bins; for each window the whole list is streamed
//                 and only in-window records are accumulated (configs 3-4).
#include <algorithm>
#include <climits>

#include "eucalc_internal.cuh"

namespace eucalc {
namespace {

constexpr unsigned long long kAgg = 1ull << 62, kIncl = 2ull << 62;
constexpr unsigned long long kM31 = (1ull << 31) - 1;

__device__ __forceinline__ unsigned long long ld_relaxed(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_relaxed(unsigned long long *p, unsigned long long v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long pack2(long long c, long long o) {
    return ((unsigned long long)c << 31) | (unsigned long long)o;
}

// Warp-wide look-back over segment flags (status | nc:31 | no:31). Returns the
// exclusive prefixes (nc, no) of segment s and publishes its inclusive prefix.
__device__ void seg_lookback(unsigned long long *flags, long long s, long long nc, long long no,
                             long long &exc_c, long long &exc_o) {
    const int lane = threadIdx.x & 31;
    long long ec = 0, eo = 0;
    if (s > 0) {
        if (lane == 0) st_relaxed(flags + s, kAgg | pack2(nc, no));
        long long j = s - 1;
        while (true) {
            long long idx = j - lane;
            unsigned long long f = kIncl;
            if (idx >= 0) {
                do { f = ld_relaxed(flags + idx); } while ((f >> 62) == 0);
            }
            unsigned incl = __ballot_sync(0xffffffffu, (f >> 62) == 2);
            int first = incl ? __ffs(incl) - 1 : 31;
            long long vc = 0, vo = 0;
            if (lane <= first) {
                vc = (long long)((f >> 31) & kM31);
                vo = (long long)(f & kM31);
            }
            for (int d = 16; d; d >>= 1) {
                vc += __shfl_xor_sync(0xffffffffu, vc, d);
                vo += __shfl_xor_sync(0xffffffffu, vo, d);
            }
            ec += vc;
            eo += vo;
            if (incl) break;
            j -= 32;
        }
    }
    if (lane == 0) st_relaxed(flags + s, kIncl | pack2(ec + nc, eo + no));
    exc_c = ec;
    exc_o = eo;
}

template <typename RecT>
__device__ __forceinline__ void decode(const RecT &r, const DirInfo &di, const K2Args &a, int &bin, int &wc,
                                       int &wj) {
    int h = 0;
#pragma unroll
    for (int k = 0; k < kMaxN; ++k)
        if (k < a.ndim) h += di.xs[k] * (int)((r.c >> a.sh[k]) & a.msk[k]);
    bin = h - di.hlo;
    const int x = r.a, y = r.b;
    wc = di.swap ? y : x;
    wj = di.swap ? (y - x) : (x - y);
}

__device__ __forceinline__ void unpack_bin(unsigned long long v, int &wc, int &wj) {
    wc = (int)(unsigned)(v & 0xffffffffull);
    wj = (int)((long long)(v - (unsigned long long)(long long)wc) >> 32);
}

template <typename OutT>
__device__ __forceinline__ void put(const StepsOut &o, long long pos, long long h, long long v) {
    reinterpret_cast<OutT *>(o.h)[pos] = (OutT)h;
    reinterpret_cast<OutT *>(o.v)[pos] = (OutT)v;
}
template <typename OutT>
__device__ __forceinline__ void put_v(const StepsOut &o, long long pos, long long v) {
    reinterpret_cast<OutT *>(o.v)[pos] = (OutT)v;
}

// Emit one 32-bin chunk held by a warp (lane <-> bin). Running totals and
// counters are warp-uniform.
template <typename OutT>
__device__ __forceinline__ void emit_chunk(const K2Args &a, int hbase, int wc, int wj, long long &e_run,
                                           long long &r_run, long long &pos_c, long long &pos_o) {
    const int lane = threadIdx.x & 31;
    int ic = wc, ij = wj;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        int tc = __shfl_up_sync(0xffffffffu, ic, d);
        int tj = __shfl_up_sync(0xffffffffu, ij, d);
        if (lane >= d) {
            ic += tc;
            ij += tj;
        }
    }
    const unsigned mc = __ballot_sync(0xffffffffu, wc != 0);
    const unsigned mo = __ballot_sync(0xffffffffu, wj != 0);
    const unsigned lt = (1u << lane) - 1;
    const long long e_incl = e_run + ic;
    const long long r_incl = r_run + ij;
    const long long h = (long long)hbase + lane;
    if (wc != 0) {
        const long long p = pos_c + __popc(mc & lt);
        if (a.do_ect) put<OutT>(a.ect, p, h, e_incl);
        if (a.do_cls) {
            if (a.cls_alias) put_v<OutT>(a.cls, p, r_incl - wj + wc);
            else put<OutT>(a.cls, p, h, r_incl - wj + wc);
        }
    }
    if (wj != 0 && a.do_ord) put<OutT>(a.ord, pos_o + __popc(mo & lt), h, r_incl);
    pos_c += __popc(mc);
    pos_o += __popc(mo);
    e_run = __shfl_sync(0xffffffffu, e_incl, 31);
    r_run = __shfl_sync(0xffffffffu, r_incl, 31);
}

__device__ __forceinline__ void write_offsets(const K2Args &a, long long s, long long exc_c, long long exc_o,
                                              long long nc, long long no) {
    const long long S = a.batch * a.D;
    if (a.do_ect) a.ect.off[s] = exc_c;
    if (a.do_cls) a.cls.off[s] = exc_c;
    if (a.do_ord) a.ord.off[s] = exc_o;
    if (s == S - 1) {
        if (a.do_ect) a.ect.off[S] = exc_c + nc;
        if (a.do_cls) a.cls.off[S] = exc_c + nc;
        if (a.do_ord) a.ord.off[S] = exc_o + no;
    }
}

// ----------------------------------------------------------------------------- warp kernel
constexpr int kWarpThreads = 256;

template <typename RecT, typename OutT>
__global__ void __launch_bounds__(kWarpThreads) k2_warp(K2Args a, int rcap, int warps, long long nblk_total,
                                                       int ndblk) {
    extern __shared__ __align__(16) unsigned long long hist_all[];
    __shared__ long long s_ticket;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    unsigned long long *hist = hist_all + (size_t)warp * rcap;
    for (int i = threadIdx.x; i < warps * rcap; i += blockDim.x) hist_all[i] = 0;
    const RecT *recs = reinterpret_cast<const RecT *>(a.rec);
    while (true) {
        __syncthreads();
        if (threadIdx.x == 0) s_ticket = (long long)atomicAdd(a.ticket, 1u);
        __syncthreads();
        const long long tk = s_ticket;
        if (tk >= nblk_total) break;
        if (warp >= warps) continue;
        const long long b = tk / ndblk;
        const long long d = (tk % ndblk) * warps + warp;
        if (d >= a.D) continue;
        const long long s = b * a.D + d;
        const DirInfo di = a.dirs[d];
        const RecT *list = recs + (b * a.Q + di.q) * a.vcap;
        const int n = a.count[b * a.Q + di.q];
        // A4: histogram (run-length merge by height)
        for (int i = lane; i < n; i += 32) {
            int bin, wc, wj;
            decode(list[i], di, a, bin, wc, wj);
            const unsigned long long pk =
                ((unsigned long long)(long long)wj << 32) + (unsigned long long)(long long)wc;
            if (pk) atomicAdd(hist + bin, pk);
        }
        __syncwarp();
        // A5 pass 1: counts
        long long nc = 0, no = 0;
        for (int base = 0; base < di.R; base += 32) {
            int wc = 0, wj = 0;
            if (base + lane < di.R) unpack_bin(hist[base + lane], wc, wj);
            nc += __popc(__ballot_sync(0xffffffffu, wc != 0));
            no += __popc(__ballot_sync(0xffffffffu, wj != 0));
        }
        long long exc_c, exc_o;
        seg_lookback(a.flags, s, nc, no, exc_c, exc_o);
        if (lane == 0) write_offsets(a, s, exc_c, exc_o, nc, no);
        // A5 pass 2: emit + clear
        long long e_run = 0, r_run = 0, pos_c = exc_c, pos_o = exc_o;
        for (int base = 0; base < di.R; base += 32) {
            int wc = 0, wj = 0;
            if (base + lane < di.R) {
                unpack_bin(hist[base + lane], wc, wj);
                hist[base + lane] = 0;
            }
            emit_chunk<OutT>(a, di.hlo + base, wc, wj, e_run, r_run, pos_c, pos_o);
        }
        __syncwarp();
    }
}

// ----------------------------------------------------------------------------- block kernel
constexpr int kBlockThreads = 512;
constexpr int kBlockWarps = kBlockThreads / 32;
constexpr int kWinBins = 26624;  // 208 KB of 64-bit bins

template <typename RecT>
__device__ void fill_window(const K2Args &a, const RecT *list, int n, const DirInfo &di, int lo, int wbins,
                            unsigned long long *hist) {
    for (int i = threadIdx.x; i < n; i += kBlockThreads) {
        int bin, wc, wj;
        decode(list[i], di, a, bin, wc, wj);
        bin -= lo;
        if ((unsigned)bin < (unsigned)wbins) {
            const unsigned long long pk =
                ((unsigned long long)(long long)wj << 32) + (unsigned long long)(long long)wc;
            if (pk) atomicAdd(hist + bin, pk);
        }
    }
}

template <typename RecT, typename OutT>
__global__ void __launch_bounds__(kBlockThreads, 1) k2_block(K2Args a, long long nseg) {
    extern __shared__ __align__(16) unsigned long long hist[];
    __shared__ long long s_seg;
    __shared__ long long s_wsum[kBlockWarps][4];  // per-warp (nc, no, sum wc, sum wj)
    __shared__ long long s_exc[2];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < kWinBins; i += kBlockThreads) hist[i] = 0;
    const RecT *recs = reinterpret_cast<const RecT *>(a.rec);
    while (true) {
        __syncthreads();
        if (threadIdx.x == 0) s_seg = (long long)atomicAdd(a.ticket, 1u);
        __syncthreads();
        const long long s = s_seg;
        if (s >= nseg) break;
        const long long b = s / a.D, d = s % a.D;
        const DirInfo di = a.dirs[d];
        const RecT *list = recs + (b * a.Q + di.q) * a.vcap;
        const int n = a.count[b * a.Q + di.q];
        const int nwin = (di.R + kWinBins - 1) / kWinBins;
        // phase A: counts over all windows
        long long nc = 0, no = 0;
        for (int w = 0; w < nwin; ++w) {
            const int lo = w * kWinBins, wb = min(kWinBins, di.R - lo);
            fill_window(a, list, n, di, lo, wb, hist);
            __syncthreads();
            int c = 0, o = 0;
            for (int i = threadIdx.x; i < wb; i += kBlockThreads) {
                int wc, wj;
                unpack_bin(hist[i], wc, wj);
                c += wc != 0;
                o += wj != 0;
                if (nwin > 1) hist[i] = 0;
            }
            for (int dd = 16; dd; dd >>= 1) {
                c += __shfl_xor_sync(0xffffffffu, c, dd);
                o += __shfl_xor_sync(0xffffffffu, o, dd);
            }
            if (lane == 0) {
                s_wsum[warp][0] = c;
                s_wsum[warp][1] = o;
            }
            __syncthreads();
            for (int k = 0; k < kBlockWarps; ++k) {
                nc += s_wsum[k][0];
                no += s_wsum[k][1];
            }
            __syncthreads();
        }
        if (warp == 0) {
            long long ec, eo;
            seg_lookback(a.flags, s, nc, no, ec, eo);
            if (lane == 0) {
                s_exc[0] = ec;
                s_exc[1] = eo;
                write_offsets(a, s, ec, eo, nc, no);
            }
        }
        __syncthreads();
        // phase B: emit, window by window; warp k owns a contiguous bin range of the window
        long long e_carry = 0, r_carry = 0, pc_carry = s_exc[0], po_carry = s_exc[1];
        for (int w = 0; w < nwin; ++w) {
            const int lo = w * kWinBins, wb = min(kWinBins, di.R - lo);
            if (nwin > 1) {
                fill_window(a, list, n, di, lo, wb, hist);
                __syncthreads();
            }
            const int per = ((wb + kBlockWarps - 1) / kBlockWarps + 31) & ~31;
            const int b0 = min(wb, warp * per), b1 = min(wb, b0 + per);
            long long c = 0, o = 0, sc = 0, sj = 0;
            for (int base = b0; base < b1; base += 32) {
                int wc = 0, wj = 0;
                if (base + lane < b1) unpack_bin(hist[base + lane], wc, wj);
                c += __popc(__ballot_sync(0xffffffffu, wc != 0));
                o += __popc(__ballot_sync(0xffffffffu, wj != 0));
                long long x = wc, y = wj;
                for (int dd = 16; dd; dd >>= 1) {
                    x += __shfl_xor_sync(0xffffffffu, x, dd);
                    y += __shfl_xor_sync(0xffffffffu, y, dd);
                }
                sc += x;
                sj += y;
            }
            if (lane == 0) {
                s_wsum[warp][0] = c;
                s_wsum[warp][1] = o;
                s_wsum[warp][2] = sc;
                s_wsum[warp][3] = sj;
            }
            __syncthreads();
            long long pc = pc_carry, po = po_carry, er = e_carry, rr = r_carry;
            long long tc = 0, to = 0, tsc = 0, tsj = 0;
            for (int k = 0; k < kBlockWarps; ++k) {
                if (k < warp) {
                    pc += s_wsum[k][0];
                    po += s_wsum[k][1];
                    er += s_wsum[k][2];
                    rr += s_wsum[k][3];
                }
                tc += s_wsum[k][0];
                to += s_wsum[k][1];
                tsc += s_wsum[k][2];
                tsj += s_wsum[k][3];
            }
            for (int base = b0; base < b1; base += 32) {
                int wc = 0, wj = 0;
                if (base + lane < b1) {
                    unpack_bin(hist[base + lane], wc, wj);
                    hist[base + lane] = 0;
                }
                emit_chunk<OutT>(a, di.hlo + lo + base, wc, wj, er, rr, pc, po);
            }
            pc_carry += tc;
            po_carry += to;
            e_carry += tsc;
            r_carry += tsj;
            __syncthreads();
        }
    }
}

template <typename RecT, typename OutT>
cudaError_t launch_t(const K2Args &a, cudaStream_t s, int num_sms) {
    const long long nseg = a.batch * a.D;
    // warp regime: whole histogram per warp, small lists
    const int rcap = (a.R_max + 31) & ~31;
    const size_t per_warp = (size_t)rcap * 8;
    int warps = (int)std::min<size_t>(8, (200 * 1024) / per_warp);
    if (warps >= 2 && a.max_count <= 32768) {
        const int ndblk = (int)((a.D + warps - 1) / warps);
        const long long nblk = a.batch * ndblk;
        const size_t smem = per_warp * warps;
        auto kern = k2_warp<RecT, OutT>;
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        int occ = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kWarpThreads, smem);
        long long grid = std::min<long long>(nblk, (long long)std::max(occ, 1) * num_sms);
        kern<<<(unsigned)grid, kWarpThreads, smem, s>>>(a, rcap, warps, nblk, ndblk);
        count_launch();
        return cudaGetLastError();
    }
    const size_t smem = (size_t)kWinBins * 8;
    auto kern = k2_block<RecT, OutT>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    long long grid = std::min<long long>(nseg, num_sms);
    kern<<<(unsigned)grid, kBlockThreads, smem, s>>>(a, nseg);
    count_launch();
    return cudaGetLastError();
}

}  // namespace

cudaError_t launch_k2(const K2Args &a, cudaStream_t s, int num_sms) {
    if (a.wide) return a.elem_bytes == 4 ? launch_t<Rec32, int32_t>(a, s, num_sms) : launch_t<Rec32, int64_t>(a, s, num_sms);
    return a.elem_bytes == 4 ? launch_t<Rec16, int32_t>(a, s, num_sms) : launch_t<Rec16, int64_t>(a, s, num_sms);
}

}  // namespace eucalc
