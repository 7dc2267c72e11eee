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
#include <type_traits>

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

// Publishes segment s's aggregate (s = 0: its inclusive prefix) for the look-backs
// of later segments (lane 0 of the calling warp).
__device__ __forceinline__ void seg_publish(unsigned long long *flags, long long s, long long nc, long long no) {
    if ((threadIdx.x & 31) == 0) st_relaxed(flags + s, (s == 0 ? kIncl : kAgg) | pack2(nc, no));
}

// Warp-wide look-back over segment flags (status | nc:31 | no:31). Returns the
// exclusive prefixes (nc, no) of segment s and publishes its inclusive prefix;
// PUBLISHED: its aggregate is already out (seg_publish).
template <bool PUBLISHED = false>
__device__ void seg_lookback(unsigned long long *flags, long long s, long long nc, long long no,
                             long long &exc_c, long long &exc_o) {
    const int lane = threadIdx.x & 31;
    long long ec = 0, eo = 0;
    if (s > 0) {
        if (!PUBLISHED && lane == 0) st_relaxed(flags + s, kAgg | pack2(nc, no));
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

// Height bin and weights of a record for direction di. DP = 2 / 3: coordinates
// are byte-aligned fields, the height is one dp2a / dp4a; DP = 0: shifts and
// masks; DP = -1: a.dp chosen at run time.
template <int DP = -1, typename RecT>
__device__ __forceinline__ void decode(const RecT &r, const DirInfo &di, const K2Args &a, int &bin, int &wc,
                                       int &wj) {
    int h = 0;
    const int dp = DP >= 0 ? DP : a.dp;
    if (dp == 2) {
        // h = sum of 16-bit unsigned coordinate halves x signed int8 direction bytes
        asm("dp2a.lo.u32.s32 %0, %1, %2, %3;" : "=r"(h) : "r"(r.c), "r"(di.xs8), "r"(-di.hlo));
        bin = h;
    } else if (dp == 3) {
        asm("dp4a.u32.s32 %0, %1, %2, %3;" : "=r"(h) : "r"(r.c), "r"(di.xs8), "r"(-di.hlo));
        bin = h;
    } else {
#pragma unroll
        for (int k = 0; k < kMaxN; ++k)
            if (k < a.ndim) h += di.xs[k] * (int)((r.c >> a.sh[k]) & a.msk[k]);
        bin = h - di.hlo;
    }
    const int x = r.a, y = r.b;
    wc = di.swap ? y : x;
    wj = di.swap ? (y - x) : (x - y);
}

// Height histogram in shared memory with native 32-bit atomics (ATOMS.ADD;
// 64-bit shared atomics are a CAS loop on sm_100a).
//   PACK : one u32 per bin holding wj * 2^16 + wc, a linear packing that is
//          exact while every bin's |sum| < 2^15 (host-checked bound).
//   SPLIT: two u32 arrays (sum Delta^-, sum J), int32 sums.
// Bin b lives in word b ^ ((b >> 5) & 31) (a permutation inside each 32-bin
// block): records streamed in vertex order hit bins in arithmetic progressions
// of stride xs_x (often a multiple of 8, 16 or 32), which without the XOR fall
// into a few of the 32 banks and serialise the atomics.
__device__ __forceinline__ int swz(int b) { return b ^ ((b >> 5) & 31); }

// SWZ: bin b lives in word swz(b) (block regime, long streams of 3-D / large
// 2-D lists); else word b, and the scan reads a lane's 4 bins with one LDS.128
// (warp regime, where the lists are short and the scan dominates).
template <bool PACK, bool SWZ = false>
struct Hist {
    unsigned *c;
    unsigned *j;
    int nb = 0x7fffffff;  // bins the arrays hold (device checks)
    __device__ __forceinline__ void add(int bin, int wc, int wj) const {
        EU_DCHECK(bin >= 0 && bin < nb);
        const int w = SWZ ? swz(bin) : bin;
        if (PACK) {
            // a kept record has Delta^-(eps) != 0 or Delta^-(-eps) != 0, so (wc, wj) != (0, 0)
            atomicAdd(c + w, (unsigned)(wj * 65536 + wc));
        } else {
            if (wc) atomicAdd(c + w, (unsigned)wc);
            if (wj) atomicAdd(j + w, (unsigned)wj);
        }
    }
    // PACK, checked: the same add, returning nonzero if the bin's new packed word
    // leaves [-2^14, 2^14) in either field. The atomic's old value is the exact sum
    // of the adds before it in the bin's atomic order; if every such prefix stayed
    // in range, one more record (|field| <= max_rec < 2^14) cannot wrap a field, so
    // the first prefix that leaves the range is decoded exactly and flagged. No flag
    // anywhere => every bin's final sums are in range and the packed words exact.
    // (x + 2^14 in both fields has bits 15 and 31 clear iff both are in range:
    // bias 0x40004000, mask 0x80008000; EUCALC_K2_CHK_BITS < 14 narrows the range
    // for tests.)
    // Returns the biased new word; the caller ORs these and tests the OR against
    // the mask once ((x & m) | (y & m) = (x | y) & m).
    __device__ __forceinline__ unsigned add_chk(int bin, int wc, int wj, unsigned bias) const {
        EU_DCHECK(bin >= 0 && bin < nb);
        const int w = SWZ ? swz(bin) : bin;
        const unsigned v = (unsigned)(wj * 65536 + wc);
        const unsigned old = atomicAdd(c + w, v);
        return old + v + bias;
    }
    // PACK only: the raw packed words of bins b0..b0+3 (b0 % 4 == 0), optionally cleared
    __device__ __forceinline__ void load4raw(int b0, unsigned (&u)[4], bool clear) const {
        if constexpr (SWZ) {
#pragma unroll
            for (int s = 0; s < 4; ++s) {
                const int w = swz(b0 + s);
                u[s] = c[w];
                if (clear) c[w] = 0;
            }
        } else {
            const uint4 v = *reinterpret_cast<const uint4 *>(c + b0);
            if (clear) *reinterpret_cast<uint4 *>(c + b0) = make_uint4(0, 0, 0, 0);
            u[0] = v.x;
            u[1] = v.y;
            u[2] = v.z;
            u[3] = v.w;
        }
    }
    // bins b0..b0+3 (b0 % 4 == 0), optionally cleared
    __device__ __forceinline__ void load4(int b0, int (&wc)[4], int (&wj)[4], bool clear) const {
        if constexpr (SWZ) {
#pragma unroll
            for (int s = 0; s < 4; ++s) {
                const int w = swz(b0 + s);
                if (PACK) {
                    const unsigned u = c[w];
                    wc[s] = (int)(short)(u & 0xffffu);
                    wj[s] = ((int)u - wc[s]) >> 16;
                } else {
                    wc[s] = (int)c[w];
                    wj[s] = (int)j[w];
                }
                if (clear) {
                    c[w] = 0;
                    if (!PACK) j[w] = 0;
                }
            }
        } else if constexpr (PACK) {
            uint4 v = *reinterpret_cast<const uint4 *>(c + b0);
            if (clear) *reinterpret_cast<uint4 *>(c + b0) = make_uint4(0, 0, 0, 0);
            const unsigned u[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int s = 0; s < 4; ++s) {
                wc[s] = (int)(short)(u[s] & 0xffffu);
                wj[s] = ((int)u[s] - wc[s]) >> 16;
            }
        } else {
            uint4 v = *reinterpret_cast<const uint4 *>(c + b0);
            uint4 w = *reinterpret_cast<const uint4 *>(j + b0);
            if (clear) {
                *reinterpret_cast<uint4 *>(c + b0) = make_uint4(0, 0, 0, 0);
                *reinterpret_cast<uint4 *>(j + b0) = make_uint4(0, 0, 0, 0);
            }
            wc[0] = (int)v.x; wc[1] = (int)v.y; wc[2] = (int)v.z; wc[3] = (int)v.w;
            wj[0] = (int)w.x; wj[1] = (int)w.y; wj[2] = (int)w.z; wj[3] = (int)w.w;
        }
    }
};

template <typename OutT>
__device__ __forceinline__ void put(const StepsOut &o, long long pos, int h, int v) {
    reinterpret_cast<OutT *>(o.h)[pos] = (OutT)h;
    reinterpret_cast<OutT *>(o.v)[pos] = (OutT)v;
}
template <typename OutT>
__device__ __forceinline__ void put_v(const StepsOut &o, long long pos, int v) {
    reinterpret_cast<OutT *>(o.v)[pos] = (OutT)v;
}

// Inclusive warp scan; the shuffle's own in-range predicate guards the add
// (2 instructions per step).
__device__ __forceinline__ int warp_incl_scan(int v) {
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        asm("{\n\t.reg .s32 t;\n\t.reg .pred p;\n\t"
            "shfl.sync.up.b32 t|p, %0, %1, 0x0, 0xffffffff;\n\t"
            "@p add.s32 %0, t, %0;\n\t}"
            : "+r"(v)
            : "r"(d));
    }
    return v;
}

// Three inclusive warp scans at once: the shuffle chains are independent, so
// interleaving them hides the shuffle latency (the emit pass was short-
// scoreboard bound on three back-to-back dependent chains).
__device__ __forceinline__ void warp_incl_scan3(int &x, int &y, int &z) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const int tx = __shfl_up_sync(0xffffffffu, x, d);
        const int ty = __shfl_up_sync(0xffffffffu, y, d);
        const int tz = __shfl_up_sync(0xffffffffu, z, d);
        if (lane >= d) {
            x += tx;
            y += ty;
            z += tz;
        }
    }
}

// Count the nonzero bins of one 128-bin group (lane <-> 4 consecutive bins).
template <bool PACK, bool SWZ>
__device__ __forceinline__ void count_group(const Hist<PACK, SWZ> &hs, int base, int &c, int &o, bool clear) {
    if constexpr (PACK) {
        // packed word u = wj * 2^16 + wc: wc != 0 <=> low half != 0; wj != 0 <=> u != sext16(u)
        unsigned u[4];
        hs.load4raw(base + 4 * (threadIdx.x & 31), u, clear);
#pragma unroll
        for (int s = 0; s < 4; ++s) {
            c += (u[s] & 0xffffu) != 0;
            o += (int)u[s] != (int)(short)(u[s] & 0xffffu);
        }
    } else {
        int wc[4], wj[4];
        hs.load4(base + 4 * (threadIdx.x & 31), wc, wj, clear);
#pragma unroll
        for (int s = 0; s < 4; ++s) {
            c += wc[s] != 0;
            o += wj[s] != 0;
        }
    }
}

// Which streams an emission writes: compile-time for the common requests,
// kModeAny checks K2Args at run time.
constexpr int kEct = 1, kOrd = 2, kCls = 4, kAlias = 8, kModeAny = 16, kHt = 32;

template <typename OutT>
struct OutPtrs {
    OutT *eh, *ev, *oh, *ov, *ch, *cv;
    const double *tab;  // fused HT (NEXT f2): kbar table over u = 2H - L*csum, or NULL
    bool ect, ord, cls, alias;
    long long cap;      // entries each array holds (device checks); staging views set their own
    __device__ explicit OutPtrs(const K2Args &a)
        : eh((OutT *)a.ect.h), ev((OutT *)a.ect.v), oh((OutT *)a.ord.h), ov((OutT *)a.ord.v),
          ch((OutT *)a.cls.h), cv((OutT *)a.cls.v), tab(a.ht_tab), ect(a.do_ect), ord(a.do_ord), cls(a.do_cls),
          alias(a.cls_alias), cap(a.out_cap) {}
};

// Fused HT (NEXT row f2): the merged histogram already holds, per lattice
// height h, H_J(h) = sum of J over the records at h, so
//   HT(xi) = -sum_x J(x) kbar(t(x)) = -sum_h H_J(h) kbar(t(h))      (Lemma 2)
// costs one table lookup per nonzero bin instead of one kbar per record.
// The table is parity-split (k3_table split = 1): u - U0 = 2h - L*csum - U0 has the
// parity of t = -L*csum - U0 for every height h of a direction, so its entries
// are contiguous: index(h) = h + tab_off with tab_off = (t & 1) * ceil(U/2) + (t >> 1).
__device__ __forceinline__ void ht_write(const K2Args &a, long long s, double acc) {
    const double v = a.ht_scale * acc;
    if (a.ht_prec == EUCALC_F32) reinterpret_cast<float *>(a.ht_out)[s] = (float)v;
    else reinterpret_cast<double *>(a.ht_out)[s] = v;
}
__device__ __forceinline__ long long ht_tab_off(const K2Args &a, const DirInfo &di) {
    const long long t = -di.lcsum - a.ht_U0;
    return (t & 1) * ((a.ht_U + 1) >> 1) + (t >> 1);
}

template <int MODE, typename OutT>
__device__ __forceinline__ void put_c(const OutPtrs<OutT> &o, int p, int h, int e, int cv) {
    EU_DCHECK(p >= 0 && p < o.cap);
    const bool ect = MODE == kModeAny ? o.ect : (MODE & kEct);
    const bool cls = MODE == kModeAny ? o.cls : (MODE & kCls);
    const bool alias = MODE == kModeAny ? o.alias : (MODE & kAlias);
    if (ect) {
        __stcs(o.eh + p, (OutT)h);
        __stcs(o.ev + p, (OutT)e);
    }
    if (cls) {
        if (!alias) __stcs(o.ch + p, (OutT)h);
        __stcs(o.cv + p, (OutT)cv);
    }
}
template <int MODE, typename OutT>
__device__ __forceinline__ void put_o(const OutPtrs<OutT> &o, int p, int h, int r) {
    EU_DCHECK(p >= 0 && p < o.cap);
    const bool ord = MODE == kModeAny ? o.ord : (MODE & kOrd);
    if (ord) {
        __stcs(o.oh + p, (OutT)h);
        __stcs(o.ov + p, (OutT)r);
    }
}

// Predicated global store (no branch: every lane computes the address; a
// divergent `if` around the store costs a reconvergence stack push/pop and the
// base pointers' reload on each side).
template <typename OutT>
__device__ __forceinline__ void st_if(OutT *p, int v, bool pred) {
    if constexpr (sizeof(OutT) == 2)
        asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t@q st.global.b16 [%0], %1;\n\t}" ::"l"(p),
                     "h"((unsigned short)v), "r"((unsigned)pred)
                     : "memory");
    else if constexpr (sizeof(OutT) == 4)
        asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t@q st.global.b32 [%0], %1;\n\t}" ::"l"(p),
                     "r"(v), "r"((unsigned)pred)
                     : "memory");
    else
        asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t@q st.global.b64 [%0], %1;\n\t}" ::"l"(p),
                     "l"((long long)v), "r"((unsigned)pred)
                     : "memory");
}
template <int MODE, typename OutT>
__device__ __forceinline__ void put_c_if(const OutPtrs<OutT> &o, int p, int h, int e, int cv, bool pred) {
    EU_DCHECK(!pred || (p >= 0 && p < o.cap));
    const bool ect = MODE == kModeAny ? o.ect : (MODE & kEct);
    const bool cls = MODE == kModeAny ? o.cls : (MODE & kCls);
    const bool alias = MODE == kModeAny ? o.alias : (MODE & kAlias);
    if (ect) {
        st_if(o.eh + p, h, pred);
        st_if(o.ev + p, e, pred);
    }
    if (cls) {
        if (!alias) st_if(o.ch + p, h, pred);
        st_if(o.cv + p, cv, pred);
    }
}
template <int MODE, typename OutT>
__device__ __forceinline__ void put_o_if(const OutPtrs<OutT> &o, int p, int h, int r, bool pred) {
    EU_DCHECK(!pred || (p >= 0 && p < o.cap));
    const bool ord = MODE == kModeAny ? o.ord : (MODE & kOrd);
    if (ord) {
        st_if(o.oh + p, h, pred);
        st_if(o.ov + p, r, pred);
    }
}

// Emit one 128-bin group held by a warp (lane <-> 4 consecutive bins) in height
// order: local sums per lane, one warp scan of (counts, sum Delta^-, sum J),
// then up to 4 entries per stream per lane. Running values are warp-uniform;
// positions are int32 (< 2^31 entries per call, host-checked).
// Two inclusive warp scans at once (see warp_incl_scan3).
__device__ __forceinline__ void warp_incl_scan2(int &x, int &y) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const int tx = __shfl_up_sync(0xffffffffu, x, d);
        const int ty = __shfl_up_sync(0xffffffffu, y, d);
        if (lane >= d) {
            x += tx;
            y += ty;
        }
    }
}

// emit_group for packed bins whose running sums fit 16 bits (every |E|, |Radon|
// <= the list's sum |a|+|b| < 2^15, host-checked; always true for int16 outputs):
// the running pair (E, Radon) is carried as ONE packed int P = Radon * 2^16 + E
// (linear, exact in int32), so the warp scans two chains instead of three, and
// E = sext16(P), Radon = (P + 2^15) >> 16. The kbar table values of the lane's
// bins are loaded before the scan so their latency overlaps it.
template <int MODE, typename OutT, bool SWZ>
__device__ __forceinline__ void emit_group16(const OutPtrs<OutT> &o, const Hist<true, SWZ> &hs, int base, int h0,
                                             int &e_run, int &r_run, int &pc, int &po, double &ht,
                                             long long tab_off) {
    const int lane = threadIdx.x & 31;
    const bool do_ht = (MODE == kModeAny) ? (o.tab != nullptr) : ((MODE & kHt) != 0);
    unsigned u[4];
    hs.load4raw(base + 4 * lane, u, true);
    const int hb = h0 + base + 4 * lane;
    int wc[4], lc = 0, lo = 0, sum = 0;
    bool nzc[4], nzo[4];
#pragma unroll
    for (int s = 0; s < 4; ++s) {
        wc[s] = (int)(short)(u[s] & 0xffffu);
        nzc[s] = wc[s] != 0;
        nzo[s] = (int)u[s] != wc[s];
        lc += nzc[s];
        lo += nzo[s];
        sum += (int)u[s];
    }
    double tv[4];
    if (do_ht) {
#pragma unroll
        for (int s = 0; s < 4; ++s) tv[s] = nzo[s] ? __ldg(o.tab + ((long long)hb + tab_off) + s) : 0.0;
    }
    const int cnt = lc | (lo << 16);
    int ic = cnt, isum = sum;
    warp_incl_scan2(ic, isum);
    const int ec = ic - cnt;
    int p_c = pc + (ec & 0xffff), p_o = po + (ec >> 16);
    const int prun = r_run * 65536 + e_run;
    int P = prun + (isum - sum);
#pragma unroll
    for (int s = 0; s < 4; ++s) {
        const int Pb = P;
        P += (int)u[s];
        put_c_if<MODE>(o, p_c, hb + s, (int)(short)(P & 0xffff), ((Pb + 0x8000) >> 16) + wc[s], nzc[s]);
        put_o_if<MODE>(o, p_o, hb + s, (P + 0x8000) >> 16, nzo[s]);
        p_c += nzc[s];
        p_o += nzo[s];
        if (do_ht && nzo[s]) ht = fma((double)(((int)u[s] - wc[s]) >> 16), tv[s], ht);
    }
    const int tc = __shfl_sync(0xffffffffu, ic, 31);
    pc += tc & 0xffff;
    po += tc >> 16;
    const int pend = prun + __shfl_sync(0xffffffffu, isum, 31);
    e_run = (int)(short)(pend & 0xffff);
    r_run = (pend + 0x8000) >> 16;
}

template <int MODE, typename OutT>
__device__ __forceinline__ void emit_words(const OutPtrs<OutT> &o, const int (&wc)[4], const int (&wj)[4], int base,
                                           int h0, int &e_run, int &r_run, int &pc, int &po, double &ht,
                                           long long tab_off);

template <int MODE, typename OutT, bool PACK, bool SWZ>
__device__ __forceinline__ void emit_group(const OutPtrs<OutT> &o, const Hist<PACK, SWZ> &hs, int base, int h0,
                                           int &e_run, int &r_run, int &pc, int &po, double &ht,
                                           long long tab_off) {
    if constexpr (PACK && sizeof(OutT) == 2) {
        emit_group16<MODE>(o, hs, base, h0, e_run, r_run, pc, po, ht, tab_off);
        return;
    }
    const int lane = threadIdx.x & 31;
    int wc[4], wj[4];
    hs.load4(base + 4 * lane, wc, wj, true);
    emit_words<MODE>(o, wc, wj, base, h0, e_run, r_run, pc, po, ht, tab_off);
}

// The emission of one 128-bin group given the lane's four bins (sum Delta^-, sum J).
template <int MODE, typename OutT>
__device__ __forceinline__ void emit_words(const OutPtrs<OutT> &o, const int (&wc)[4], const int (&wj)[4], int base,
                                           int h0, int &e_run, int &r_run, int &pc, int &po, double &ht,
                                           long long tab_off) {
    const int lane = threadIdx.x & 31;
    int lc = 0, lo = 0, sc = 0, sj = 0;
#pragma unroll
    for (int s = 0; s < 4; ++s) {
        lc += wc[s] != 0;
        lo += wj[s] != 0;
        sc += wc[s];
        sj += wj[s];
    }
    const int cnt = lc | (lo << 16);
    int ic = cnt, isc = sc, isj = sj;
    warp_incl_scan3(ic, isc, isj);
    const int ec = ic - cnt;
    int p_c = pc + (ec & 0xffff), p_o = po + (ec >> 16);
    int e = e_run + (isc - sc), r = r_run + (isj - sj);
    const int hb = h0 + base + 4 * lane;
#pragma unroll
    for (int s = 0; s < 4; ++s) {
        const int rb = r;
        e += wc[s];
        r += wj[s];
        if (wc[s]) put_c<MODE>(o, p_c++, hb + s, e, rb + wc[s]);
        if (wj[s]) put_o<MODE>(o, p_o++, hb + s, r);
        const bool do_ht = (MODE == kModeAny) ? (o.tab != nullptr) : ((MODE & kHt) != 0);
        if (do_ht && wj[s]) ht = fma((double)wj[s], __ldg(o.tab + (long long)(hb + s) + tab_off), ht);
    }
    const int tc = __shfl_sync(0xffffffffu, ic, 31);
    pc += tc & 0xffff;
    po += tc >> 16;
    e_run += __shfl_sync(0xffffffffu, isc, 31);
    r_run += __shfl_sync(0xffffffffu, isj, 31);
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

__device__ __forceinline__ int warp_sum(int v) {
#pragma unroll
    for (int d = 16; d; d >>= 1) v += __shfl_xor_sync(0xffffffffu, v, d);
    return v;
}

// ----------------------------------------------------------------------------- warp kernel
constexpr int kWarpThreads = 256;
constexpr int kGroup = 128;  // bins per warp step (4 per lane)

// Warp regime, three launches with no cross-segment waiting:
//   k2w_count: per segment (one warp, dynamic ticket) histogram + count of the
//              nonzero bins of each stream -> counts[s] (the histogram is
//              cleared while counting);
//   k2_scan  : exclusive scan of the counts -> CSR offsets;
//   k2w_emit : per segment histogram again + ordered emission at its offset.
// (A single pass with a segment look-back was measured to lose ~1/3 of the
// time to look-back spinning when ~9k warps start at once.)
// Packed bin word of a 16-bit record for the direction's orthant, from the
// record's weight word w = a | b << 16: wj * 2^16 + wc with (wc, wj) = (a, a - b)
// (representative orthant) or (b, b - a) (its antipode, SWAP): one extract, one
// mask/shift, one multiply-add.
template <bool SWAP>
__device__ __forceinline__ unsigned packed_word(unsigned w) {
    if (SWAP) return (unsigned)(((int)w >> 16) * 65537 - (int)(w << 16));
    return (unsigned)((int)(short)(w & 0xffffu) * 65537 - (int)(w & 0xffff0000u));
}

template <int DP, bool SWAP, typename RecT, bool PACK>
__device__ __forceinline__ void fill_loop(const K2Args &a, const Hist<PACK> &hs, const RecT *list, int n,
                                          const DirInfo &di, int &lo, int &hi) {
    const int lane = threadIdx.x & 31;
    int i = lane;
    for (; i + 32 < n; i += 64) {  // two records in flight per lane
        const RecT r0 = list[i], r1 = list[i + 32];
        int bin0, wc0, wj0, bin1, wc1, wj1;
        decode<DP>(r0, di, a, bin0, wc0, wj0);
        decode<DP>(r1, di, a, bin1, wc1, wj1);
        if constexpr (PACK && std::is_same<RecT, Rec16>::value) {
            EU_DCHECK(bin0 >= 0 && bin0 < hs.nb && bin1 >= 0 && bin1 < hs.nb);
            atomicAdd(hs.c + bin0, packed_word<SWAP>(reinterpret_cast<const uint2 &>(r0).y));
            atomicAdd(hs.c + bin1, packed_word<SWAP>(reinterpret_cast<const uint2 &>(r1).y));
        } else {
            hs.add(bin0, wc0, wj0);
            hs.add(bin1, wc1, wj1);
        }
        lo = min(lo, min(bin0, bin1));
        hi = max(hi, max(bin0, bin1));
    }
    if (i < n) {
        const RecT r = list[i];
        int bin, wc, wj;
        decode<DP>(r, di, a, bin, wc, wj);
        if constexpr (PACK && std::is_same<RecT, Rec16>::value) {
            EU_DCHECK(bin >= 0 && bin < hs.nb);
            atomicAdd(hs.c + bin, packed_word<SWAP>(reinterpret_cast<const uint2 &>(r).y));
        }
        else
            hs.add(bin, wc, wj);
        lo = min(lo, bin);
        hi = max(hi, bin);
    }
}

template <typename RecT, bool PACK>
// Fills the warp's histogram with the segment's records; returns the 128-bin
// groups [g0, g1) that can hold a nonzero bin (the records' height span,
// typically ~85% of R: the scans skip the rest). The loop is specialised on the
// height decode and the orthant side (both uniform per segment).
__device__ __forceinline__ void fill_segment(const K2Args &a, const Hist<PACK> &hs, long long b, const DirInfo &di,
                                             int &g0, int &g1) {
    const RecT *list = reinterpret_cast<const RecT *>(a.rec) + (b * a.Q + di.q) * a.vcap;
    const int n = a.count[b * a.Q + di.q];
    int lo = INT_MAX, hi = -1;
    if (a.dp == 2) {
        if (di.swap) fill_loop<2, true>(a, hs, list, n, di, lo, hi);
        else fill_loop<2, false>(a, hs, list, n, di, lo, hi);
    } else if (a.dp == 3) {
        if (di.swap) fill_loop<3, true>(a, hs, list, n, di, lo, hi);
        else fill_loop<3, false>(a, hs, list, n, di, lo, hi);
    } else {
        if (di.swap) fill_loop<0, true>(a, hs, list, n, di, lo, hi);
        else fill_loop<0, false>(a, hs, list, n, di, lo, hi);
    }
    for (int d = 16; d; d >>= 1) {
        lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, d));
        hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, d));
    }
    g0 = hi < 0 ? 0 : (lo / kGroup) * kGroup;
    g1 = hi + 1;
    __syncwarp();
}

// Sparse path for lists of <= 32 records (e.g. binary images): the records'
// (height, Delta^-, J) are sorted across the warp by a register bitonic
// network and equal heights merged by prefix sums — the paper's sort +
// merge without touching R bins.
struct SparseRuns {
    int h;            // bin (height - hlo) of this lane's sorted record
    int pc, pj;       // inclusive prefix sums of Delta^- and J in sorted order
    int run_c, run_j; // sums over this lane's equal-height run (valid at run ends)
    bool emit_c, emit_o;
};

// Bitonic network over the first KMAX lanes (fully unrolled: every step a
// compile-time shuffle distance and a per-lane min/max choice).
template <int KMAX>
__device__ __forceinline__ int bitonic_keys(int key) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int k = 2; k <= KMAX; k <<= 1) {
#pragma unroll
        for (int j = k >> 1; j > 0; j >>= 1) {
            const int ok = __shfl_xor_sync(0xffffffffu, key, j);
            const bool takemin = ((lane & j) == 0) == ((lane & k) == 0);
            key = takemin ? min(key, ok) : max(key, ok);
        }
    }
    return key;
}

template <typename RecT>
__device__ __forceinline__ SparseRuns sparse_runs(const K2Args &a, long long b, const DirInfo &di, int n) {
    const int lane = threadIdx.x & 31;
    const RecT *list = reinterpret_cast<const RecT *>(a.rec) + (b * a.Q + di.q) * a.vcap;
    int h = 0, wc = 0, wj = 0;
    if (lane < n) decode(list[lane], di, a, h, wc, wj);
    // Sort the keys (bin << 5 | lane) — unique, so one shuffle and one min/max per
    // network step; padding lanes hold keys above every record's. A list of
    // <= 16 (8) records is sorted by the 16 (8)-lane network (the padding lanes
    // above it are already in order).
    int key = lane < n ? (h << 5) | lane : (0x7fffffe0 | lane);
    if (n <= 8) key = bitonic_keys<8>(key);
    else if (n <= 16) key = bitonic_keys<16>(key);
    else key = bitonic_keys<32>(key);
    const int src = key & 31;
    const bool valid = key < 0x7fffffe0;
    SparseRuns r;
    r.h = valid ? key >> 5 : INT_MAX;
    if (a.sum16) {
        // one scan of the packed pair (|prefix sums| <= list sum |a|+|b| < 2^15)
        const int w = __shfl_sync(0xffffffffu, wj * 65536 + wc, src);
        const int pw = warp_incl_scan(valid ? w : 0);
        r.pc = (int)(short)(pw & 0xffff);
        r.pj = (pw + 0x8000) >> 16;
    } else {
        wc = __shfl_sync(0xffffffffu, wc, src);
        wj = __shfl_sync(0xffffffffu, wj, src);
        r.pc = warp_incl_scan(valid ? wc : 0);
        r.pj = warp_incl_scan(valid ? wj : 0);
    }
    const int hn = __shfl_down_sync(0xffffffffu, r.h, 1);
    const int hp = __shfl_up_sync(0xffffffffu, r.h, 1);
    const bool end = lane == 31 || hn != r.h;
    const bool head = lane == 0 || hp != r.h;
    // run start: the highest head lane <= this lane
    const unsigned heads = __ballot_sync(0xffffffffu, head);
    const int st = 31 - __clz(heads & (0xffffffffu >> (31 - lane)));
    const int bsrc = st > 0 ? st - 1 : 0;
    const int bc = __shfl_sync(0xffffffffu, r.pc, bsrc), bj = __shfl_sync(0xffffffffu, r.pj, bsrc);
    r.run_c = r.pc - (st > 0 ? bc : 0);
    r.run_j = r.pj - (st > 0 ? bj : 0);
    r.emit_c = end && valid && r.run_c != 0;
    r.emit_o = end && valid && r.run_j != 0;
    return r;
}

template <bool PACK>
__device__ __forceinline__ Hist<PACK> warp_hist(unsigned *smem, int rcap) {
    constexpr int words = PACK ? 1 : 2;
    const int warp = threadIdx.x >> 5;
    Hist<PACK> hs;
    hs.c = smem + (size_t)warp * rcap * words;
    hs.j = hs.c + rcap;
    hs.nb = rcap;
    for (int i = threadIdx.x; i < (int)(blockDim.x / 32) * rcap * words; i += blockDim.x) smem[i] = 0;
    __syncthreads();
    return hs;
}


template <typename RecT, bool PACK>
__global__ void __launch_bounds__(kWarpThreads) k2w_count(K2Args a, int rcap, int *cnt_c, int *cnt_o) {
    extern __shared__ __align__(16) unsigned hist_all[];
    const Hist<PACK> hs = warp_hist<PACK>(hist_all, rcap);
    // segment indices are int32 (< 2^31 segments per call, host-checked): no 64-bit division
    const int S = (int)(a.batch * a.D), D = (int)a.D;
    const int nw = gridDim.x * (blockDim.x >> 5);
    const int s0 = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int nb = nw / D, nd = nw - nb * D;  // (image, direction) advance per step
    int b = s0 / D, d = s0 - b * D;
    for (int s = s0; s < S; s += nw, b += nb, d += nd) {
        if (d >= D) {
            d -= D;
            ++b;
        }
        const DirInfo di = a.dirs[d];
        const int n = a.count[b * a.Q + di.q];
        int c = 0, o = 0;
        if (n <= a.sparse_max) {
            const SparseRuns r = sparse_runs<RecT>(a, b, di, n);
            const unsigned mc = __ballot_sync(0xffffffffu, r.emit_c), mo = __ballot_sync(0xffffffffu, r.emit_o);
            c = __popc(mc);
            o = __popc(mo);
            if (a.slab) {
                // keep the merged runs for k2w_emit (16-bit fields, host-checked):
                // bin | E << 16, E_c | E' << 16; the emission masks in slot 32
                const int ec = r.pj - r.run_j + r.run_c;
                uint2 *sl = a.slab + (long long)s * 33;
                sl[threadIdx.x & 31] = make_uint2((unsigned)(r.h & 0xffff) | ((unsigned)r.pc << 16),
                                                  (unsigned)(ec & 0xffff) | ((unsigned)r.pj << 16));
                if ((threadIdx.x & 31) == 0) sl[32] = make_uint2(mc, mo);
            }
            if (a.ht_tab) {
                // fused HT of a sparse segment: one term per merged run (fixed-order tree sum)
                double acc = 0.0;
                if (r.emit_o) acc = (double)r.run_j * __ldg(a.ht_tab + (long long)(di.hlo + r.h) + ht_tab_off(a, di));
                for (int k = 16; k; k >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, k);
                if ((threadIdx.x & 31) == 0) ht_write(a, s, acc);
            }
        } else {
            int g0, g1;
            fill_segment<RecT>(a, hs, b, di, g0, g1);
            for (int base = g0; base < g1; base += kGroup) count_group(hs, base, c, o, true);
            c = warp_sum(c);
            o = warp_sum(o);
        }
        if ((threadIdx.x & 31) == 0) {
            cnt_c[s] = c;
            cnt_o[s] = o;
        }
        __syncwarp();
    }
}

template <typename RecT, typename OutT, bool PACK, int MODE>
__global__ void __launch_bounds__(kWarpThreads, 5) k2w_emit(K2Args a, int rcap) {
    extern __shared__ __align__(16) unsigned hist_all[];
    const Hist<PACK> hs = warp_hist<PACK>(hist_all, rcap);
    const OutPtrs<OutT> o(a);
    const int S = (int)(a.batch * a.D), D = (int)a.D;
    const int64_t *off_c = a.do_ect ? a.ect.off : a.cls.off;
    const bool any_c = a.do_ect || a.do_cls;
    const int nw = gridDim.x * (blockDim.x >> 5);
    const int s0 = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int nb = nw / D, nd = nw - nb * D;  // (image, direction) advance per step
    int b = s0 / D, d = s0 - b * D;
    for (int s = s0; s < S; s += nw, b += nb, d += nd) {
        if (d >= D) {
            d -= D;
            ++b;
        }
        const DirInfo di = a.dirs[d];
        const int n = a.count[b * a.Q + di.q];
        int pc = any_c ? (int)off_c[s] : 0, po = a.do_ord ? (int)a.ord.off[s] : 0;
        if (n <= a.sparse_max) {
            const unsigned lt = (1u << (threadIdx.x & 31)) - 1;
            if (a.slab) {
                const uint2 *sl = a.slab + (long long)s * 33;
                const uint2 v = sl[threadIdx.x & 31], m = sl[32];
                const int h = di.hlo + (int)(v.x & 0xffff);
                const int e = (int)v.x >> 16, ec = (int)(short)(v.y & 0xffff), eo = (int)v.y >> 16;
                if ((m.x >> (threadIdx.x & 31)) & 1) put_c<MODE>(o, pc + __popc(m.x & lt), h, e, ec);
                if ((m.y >> (threadIdx.x & 31)) & 1) put_o<MODE>(o, po + __popc(m.y & lt), h, eo);
            } else {
                const SparseRuns r = sparse_runs<RecT>(a, b, di, n);
                const unsigned mc = __ballot_sync(0xffffffffu, r.emit_c), mo = __ballot_sync(0xffffffffu, r.emit_o);
                const int h = di.hlo + r.h;
                // classical value: Radon(h-) + sum Delta^- at h
                if (r.emit_c) put_c<MODE>(o, pc + __popc(mc & lt), h, r.pc, r.pj - r.run_j + r.run_c);
                if (r.emit_o) put_o<MODE>(o, po + __popc(mo & lt), h, r.pj);
            }
        } else {
            int g0, g1;
            fill_segment<RecT>(a, hs, b, di, g0, g1);
            int e_run = 0, r_run = 0;
            double ht = 0.0;
            const long long toff = (MODE & kHt) || (MODE == kModeAny && o.tab) ? ht_tab_off(a, di) : 0;
            for (int base = g0; base < g1; base += kGroup)
                emit_group<MODE>(o, hs, base, di.hlo, e_run, r_run, pc, po, ht, toff);
            if ((MODE & kHt) || (MODE == kModeAny && o.tab)) {
                for (int k = 16; k; k >>= 1) ht += __shfl_xor_sync(0xffffffffu, ht, k);
                if ((threadIdx.x & 31) == 0) ht_write(a, s, ht);
            }
        }
        __syncwarp();
    }
}

// Single-pass exclusive scan of (cnt_c, cnt_o) into the CSR offset arrays
// (tiles of 8192 counts, decoupled look-back between the few tiles).
constexpr int kScanThreads = 256, kScanPer = 8, kScanTile = kScanThreads * kScanPer;

__global__ void __launch_bounds__(kScanThreads) k2_scan(K2Args a, const int *cnt_c, const int *cnt_o, long long S,
                                                       unsigned long long *flags) {
    __shared__ long long s_w[kScanThreads / 32][2];
    __shared__ long long s_base[2];
    __shared__ unsigned s_tile;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) s_tile = atomicAdd(a.ticket + 2, 1u);
    __syncthreads();
    const long long t = s_tile;
    const long long i0 = t * kScanTile + (long long)threadIdx.x * kScanPer;
    long long lc[kScanPer], lo[kScanPer], tc = 0, to = 0;
#pragma unroll
    for (int k = 0; k < kScanPer; ++k) {
        const long long i = i0 + k;
        lc[k] = i < S ? cnt_c[i] : 0;
        lo[k] = i < S ? cnt_o[i] : 0;
        tc += lc[k];
        to += lo[k];
    }
    // block exclusive scan of thread totals
    long long ic = tc, io = to;
    for (int d = 1; d < 32; d <<= 1) {
        long long x = __shfl_up_sync(0xffffffffu, ic, d), y = __shfl_up_sync(0xffffffffu, io, d);
        if (lane >= d) { ic += x; io += y; }
    }
    if (lane == 31) { s_w[warp][0] = ic; s_w[warp][1] = io; }
    __syncthreads();
    if (warp == 0) {
        constexpr int W = kScanThreads / 32;
        long long wc = lane < W ? s_w[lane][0] : 0, wo = lane < W ? s_w[lane][1] : 0;
        long long xc = wc, xo = wo;
        for (int d = 1; d < 32; d <<= 1) {
            long long x = __shfl_up_sync(0xffffffffu, xc, d), y = __shfl_up_sync(0xffffffffu, xo, d);
            if (lane >= d) { xc += x; xo += y; }
        }
        if (lane < W) {
            s_w[lane][0] = xc - wc;
            s_w[lane][1] = xo - wo;
        }
        const long long aggc = __shfl_sync(0xffffffffu, xc, 31), aggo = __shfl_sync(0xffffffffu, xo, 31);
        long long ec, eo;
        seg_lookback(flags, t, aggc, aggo, ec, eo);
        if (lane == 0) { s_base[0] = ec; s_base[1] = eo; }
    }
    __syncthreads();
    long long pc = s_base[0] + s_w[warp][0] + ic - tc, po = s_base[1] + s_w[warp][1] + io - to;
#pragma unroll
    for (int k = 0; k < kScanPer; ++k) {
        const long long i = i0 + k;
        if (i <= S) {
            if (a.do_ect) a.ect.off[i] = pc;
            if (a.do_cls) a.cls.off[i] = pc;
            if (a.do_ord) a.ord.off[i] = po;
        }
        pc += lc[k];
        po += lo[k];
    }
}

// ----------------------------------------------------------------------------- block kernel
constexpr int kBlockThreads = 1024;
constexpr int kBlockWarps = kBlockThreads / 32;
constexpr size_t kBlockSmem = 200 * 1024;

// Accumulate the records list[beg, end) whose bin lies in [lo, lo + wbins):
// the warp's lanes stride the range, four records in flight per lane (the list
// streams from L2; a lone load per lane leaves the SM latency-bound).
// U: records in flight per thread; DP as decode; CHECK: skip records outside
// the window (false when the window covers the whole height range); CHK: checked
// packed adds (Hist::add_chk), biased words OR-ed into `bad`.
template <int U, int DP, bool CHECK, bool CHK, typename RecT, bool PACK, bool SWZ>
__device__ __forceinline__ void fill_range_t(const K2Args &a, const RecT *list, int beg, int end, const DirInfo &di,
                                             int lo, int wbins, const Hist<PACK, SWZ> &hs, int lane, int step,
                                             unsigned &bad) {
    int i = beg + lane;
    for (; i + (U - 1) * step < end; i += U * step) {
        RecT r[U];
#pragma unroll
        for (int u = 0; u < U; ++u) r[u] = list[i + u * step];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            int bin, wc, wj;
            decode<DP>(r[u], di, a, bin, wc, wj);
            bin -= lo;
            if (!CHECK || (unsigned)bin < (unsigned)wbins) {
                if constexpr (CHK) bad |= hs.add_chk(bin, wc, wj, a.chk_bias);
                else hs.add(bin, wc, wj);
            }
        }
    }
    for (; i < end; i += step) {
        int bin, wc, wj;
        decode<DP>(list[i], di, a, bin, wc, wj);
        bin -= lo;
        if (!CHECK || (unsigned)bin < (unsigned)wbins) {
            if constexpr (CHK) bad |= hs.add_chk(bin, wc, wj, a.chk_bias);
            else hs.add(bin, wc, wj);
        }
    }
}

// CHK: checked adds when `chk` (run-time uniform: a segment whose packed bins are
// proven exact skips the check and the atomics' return values).
template <int U, int DP, bool CHK, typename RecT, bool PACK, bool SWZ>
__device__ __forceinline__ void fill_range(const K2Args &a, const RecT *list, int beg, int end, const DirInfo &di,
                                           int lo, int wbins, const Hist<PACK, SWZ> &hs, int lane, int step,
                                           unsigned &bad, bool chk) {
    const bool whole = lo == 0 && wbins >= di.R;
    if (CHK && chk) {
        if (whole) fill_range_t<U, DP, false, CHK>(a, list, beg, end, di, lo, wbins, hs, lane, step, bad);
        else fill_range_t<U, DP, true, CHK>(a, list, beg, end, di, lo, wbins, hs, lane, step, bad);
    } else {
        if (whole) fill_range_t<U, DP, false, false>(a, list, beg, end, di, lo, wbins, hs, lane, step, bad);
        else fill_range_t<U, DP, true, false>(a, list, beg, end, di, lo, wbins, hs, lane, step, bad);
    }
}

// Height range (bins relative to hlo) of K1 tile t: a TZ x TY x TX box of
// vertices, so the range is sum_k min/max of xs_k times the box's extent on axis k.
__device__ __forceinline__ void tile_bins(const K2Args &a, const DirInfo &di, int t, int &bmin, int &bmax) {
    const int tx = t % a.tiles_x, ty = (t / a.tiles_x) % a.tiles_y, tz = t / (a.tiles_x * a.tiles_y);
    const int n = a.ndim;
    int lo3[kMaxN], hi3[kMaxN];
    lo3[n - 1] = tx * a.TX;
    hi3[n - 1] = min(lo3[n - 1] + a.TX, a.M[n - 1]) - 1;
    lo3[n - 2] = ty * a.TY;
    hi3[n - 2] = min(lo3[n - 2] + a.TY, a.M[n - 2]) - 1;
    if (n == 3) {
        lo3[0] = tz * a.TZ;
        hi3[0] = min(lo3[0] + a.TZ, a.M[0]) - 1;
    }
    int hmin = 0, hmax = 0;
#pragma unroll
    for (int k = 0; k < kMaxN; ++k) {
        if (k < n) {
            const int x0 = di.xs[k] * lo3[k], x1 = di.xs[k] * hi3[k];
            hmin += min(x0, x1);
            hmax += max(x0, x1);
        }
    }
    bmin = hmin - di.hlo;
    bmax = hmax - di.hlo;
}

__device__ __forceinline__ void red_smem(unsigned addr, unsigned v) {
    asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(addr), "r"(v));
}
__device__ __forceinline__ unsigned atom_smem(unsigned addr, unsigned v) {
    unsigned old;
    asm volatile("atom.shared.add.u32 %0, [%1], %2;" : "=r"(old) : "r"(addr), "r"(v));
    return old;
}

// Span fill (8-byte records, packed swizzled bins, byte-aligned coordinates): the
// list ranges ("runs") to stream are cut into chunks of kSpanChunk records, dealt
// round-robin to the warps; a lane keeps eight 8-byte loads in flight, and a record
// costs one weight word (packed_word), one dp2a/dp4a (bin relative to the window),
// the window test (CHECK), the bank swizzle and one shared atomic (CHK: checked, the
// returned word biased and OR-ed into the result). Runs come from shared tables
// (s_rb/s_re = record range, s_cpre = exclusive chunk prefix, nruns + 1 entries),
// or, nruns == 0, the single run [0, n).
constexpr int kSpanTiles = 2048;  // tiles whose hit mask and run tables fit BlockShared::hit
constexpr int kSpanChunk = 512;   // records per warp work item

template <int DP, bool CHK>
__device__ __forceinline__ unsigned span_fill(const uint2 *list, const int *s_rb, const int *s_re, const int *s_cpre,
                                              int nruns, int n, const DirInfo &di, int lo, int wb, unsigned sb,
                                              unsigned bias, int nb, int nmax) {
    constexpr int U = 8;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int xs8 = di.xs8, nhlo = -(di.hlo + lo);
    // the window test also serves a window that covers the whole range (always true);
    // the antipodal side swaps the record's two 16-bit weights before packed_word
    const unsigned wbins = (unsigned)wb, sel = di.swap ? 0x1032u : 0x3210u;
    __shared__ unsigned span_dummy[32];
    // shared addresses and the byte selector as opaque registers (else the compiler
    // rematerialises them from the CTA's shared window per record)
    unsigned dummy = (unsigned)__cvta_generic_to_shared(span_dummy) + 4u * lane, sbr = sb, selr = sel;
    asm volatile("mov.u32 %0, %0;" : "+r"(dummy));
    asm volatile("mov.u32 %0, %0;" : "+r"(sbr));
    asm volatile("mov.u32 %0, %0;" : "+r"(selr));
    unsigned bad = 0;
    auto one = [&](const uint2 r) {
        const unsigned w = packed_word<false>(__byte_perm(r.y, 0u, selr));
        int h;
        if (DP == 2) asm("dp2a.lo.u32.s32 %0, %1, %2, %3;" : "=r"(h) : "r"(r.x), "r"(xs8), "r"(nhlo));
        else asm("dp4a.u32.s32 %0, %1, %2, %3;" : "=r"(h) : "r"(r.x), "r"(xs8), "r"(nhlo));
        // no branch: a record outside the window adds 0 to the lane's own dummy word
        // (its biased word has no flag bit: bias + 0 + 0)
        const bool in = (unsigned)h < wbins;
        const unsigned addr = in ? sbr + ((unsigned)swz(h) << 2) : dummy;
        const unsigned wv = in ? w : 0u;
        if constexpr (CHK) bad |= atom_smem(addr, wv) + wv + bias;
        else red_smem(addr, wv);
    };
    const bool single = nruns == 0;
    const int total = single ? (n + kSpanChunk - 1) / kSpanChunk : s_cpre[nruns];
    int r = 0;
    for (int k = warp; k < total; k += kBlockWarps) {
        int b, e;
        if (single) {
            b = k * kSpanChunk;
            e = min(b + kSpanChunk, n);
        } else {
            while (k >= s_cpre[r + 1]) ++r;
            b = s_rb[r] + (k - s_cpre[r]) * kSpanChunk;
            e = min(b + kSpanChunk, s_re[r]);
        }
        EU_DCHECK(b >= 0 && b <= e && e <= nmax && wb <= nb);
        for (int i = b + lane; i < e; i += U * 32) {
            uint2 v[U];
            if (i + (U - 1) * 32 < e) {
#pragma unroll
                for (int u = 0; u < U; ++u) v[u] = __ldg(list + i + u * 32);
#pragma unroll
                for (int u = 0; u < U; ++u) one(v[u]);
            } else {
#pragma unroll
                for (int u = 0; u < U; ++u)
                    if (i + u * 32 < e) v[u] = __ldg(list + i + u * 32);
#pragma unroll
                for (int u = 0; u < U; ++u)
                    if (i + u * 32 < e) one(v[u]);
            }
        }
    }
    return bad;
}

// One height window of a segment: every record whose bin is in [lo, lo+wbins).
// A single window takes the whole list; several windows cull K1 tiles by their
// height band, so each record is streamed about once over all windows instead
// of once per window.
constexpr int kMaxHitTiles = 4096;  // culled-tile list in shared memory

template <int DP, bool CHK, typename RecT, bool PACK, bool SWZ>
__device__ void fill_window(const K2Args &a, const RecT *list, const int32_t *toff, int n, const DirInfo &di,
                            int lo, int wbins, bool cull, const Hist<PACK, SWZ> &hs, int *s_hit, int *s_nhit,
                            unsigned &bad, bool chk) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if constexpr (PACK && SWZ && std::is_same<RecT, Rec16>::value && (DP == 2 || DP == 3)) {
        if (!cull || a.ntiles <= kSpanTiles) {
            // span path: maximal runs of consecutive hit tiles are contiguous list ranges
            // (tile t's records are list[toff[t], toff[t+1])), streamed in warp chunks
            const uint2 *l2 = reinterpret_cast<const uint2 *>(list);
            const unsigned sb = (unsigned)__cvta_generic_to_shared(hs.c);
            int *s_mask = s_hit, *s_rb = s_hit + kSpanTiles / 32, *s_re = s_rb + kSpanTiles / 2 + 1,
                *s_cpre = s_re + kSpanTiles / 2 + 1;
            int nruns = 0;
            if (cull) {
                const int nw = (a.ntiles + 31) >> 5;
                if (threadIdx.x == 0) *s_nhit = 0;
                for (int t = threadIdx.x; t < nw * 32; t += kBlockThreads) {
                    bool hit = false;
                    if (t < a.ntiles) {
                        int bmin, bmax;
                        tile_bins(a, di, t, bmin, bmax);
                        hit = bmax >= lo && bmin < lo + wbins;
                    }
                    const unsigned m = __ballot_sync(0xffffffffu, hit);
                    if (lane == 0) s_mask[t >> 5] = (int)m;
                }
                __syncthreads();
                for (int t = threadIdx.x; t < a.ntiles; t += kBlockThreads) {
                    const unsigned m = (unsigned)s_mask[t >> 5];
                    bool start = (m >> (t & 31)) & 1u;
                    if (start && t > 0) start = !(((unsigned)s_mask[(t - 1) >> 5] >> ((t - 1) & 31)) & 1u);
                    if (start) {
                        int w = t >> 5;
                        unsigned z = ~m & (0xffffffffu << (t & 31));  // first tile after t that is not hit
                        while (!z && ++w < nw) z = ~(unsigned)s_mask[w];
                        const int e = z ? min((w << 5) + __ffs(z) - 1, a.ntiles) : a.ntiles;
                        const int rb = toff[t], re = toff[e];
                        if (re > rb) {
                            const int k = atomicAdd(s_nhit, 1);
                            EU_DCHECK(k <= kSpanTiles / 2);
                            s_rb[k] = rb;
                            s_re[k] = re;
                        }
                    }
                }
                __syncthreads();
                nruns = *s_nhit;
                if (warp == 0) {
                    int run = 0;
                    for (int base = 0; base < nruns; base += 32) {
                        const int c = base + lane < nruns
                                          ? (s_re[base + lane] - s_rb[base + lane] + kSpanChunk - 1) / kSpanChunk : 0;
                        int inc = c;
                        for (int k = 1; k < 32; k <<= 1) {
                            const int y = __shfl_up_sync(0xffffffffu, inc, k);
                            if (lane >= k) inc += y;
                        }
                        if (base + lane < nruns) s_cpre[base + lane] = run + inc - c;
                        run += __shfl_sync(0xffffffffu, inc, 31);
                    }
                    if (lane == 0) s_cpre[nruns] = run;
                }
                __syncthreads();
                if (nruns == 0) return;
            }
            if (CHK && chk) bad |= span_fill<DP, true>(l2, s_rb, s_re, s_cpre, nruns, n, di, lo, wbins, sb, a.chk_bias, hs.nb, n);
            else span_fill<DP, false>(l2, s_rb, s_re, s_cpre, nruns, n, di, lo, wbins, sb, 0u, hs.nb, n);
            return;
        }
    }
    if (!cull) {
        fill_range<8, DP, CHK>(a, list, 0, n, di, lo, wbins, hs, threadIdx.x, kBlockThreads, bad, chk);
        return;
    }
    if (a.ntiles <= kMaxHitTiles) {
        // the tiles whose height band meets the window, compacted (any order: the
        // histogram sums are integers), then dealt round-robin to the warps
        if (threadIdx.x == 0) *s_nhit = 0;
        __syncthreads();
        for (int t = threadIdx.x; t < a.ntiles; t += kBlockThreads) {
            int bmin, bmax;
            tile_bins(a, di, t, bmin, bmax);
            if (bmax >= lo && bmin < lo + wbins && toff[t + 1] > toff[t]) s_hit[atomicAdd(s_nhit, 1)] = t;
        }
        __syncthreads();
        const int nhit = *s_nhit;
        for (int k = warp; k < nhit; k += kBlockWarps) {
            const int tt = s_hit[k];
            fill_range<4, DP, CHK>(a, list, toff[tt], toff[tt + 1], di, lo, wbins, hs, lane, 32, bad, chk);
        }
        return;
    }
    for (int t0 = warp * 32; t0 < a.ntiles; t0 += kBlockWarps * 32) {
        const int t = t0 + lane;
        bool hit = false;
        if (t < a.ntiles) {
            int bmin, bmax;
            tile_bins(a, di, t, bmin, bmax);
            hit = bmax >= lo && bmin < lo + wbins;
        }
        unsigned m = __ballot_sync(0xffffffffu, hit);
        while (m) {
            const int tt = t0 + __ffs(m) - 1;
            m &= m - 1;
            fill_range<4, DP, CHK>(a, list, toff[tt], toff[tt + 1], di, lo, wbins, hs, lane, 32, bad, chk);
        }
    }
}

struct BlockShared {
    long long seg;
    int cnt[2];                // staged segment: (nc, no)
    int wsum[kBlockWarps][4];  // per-warp (nc, no, sum wc, sum wj)
    long long exc[2];
    double ht[kBlockWarps];
    int hit[kMaxHitTiles];
    int nhit;
};

// One segment (image b, direction d) of the block regime with histogram bins of
// kind PACK over windows of `win` bins (`hist` holds win words per array).
// PACK: every fill checks its adds (Hist::add_chk) against chk_mask (0 when a
// bound proves the packed bins exact); on a flag, before anything of the segment
// reaches global memory, it returns false (the caller reruns the segment with
// split bins); else true.
template <bool PACK, int DP, typename RecT, typename OutT>
__device__ __forceinline__ bool block_segment(const K2Args &a, const OutPtrs<OutT> &outp, unsigned *hist, int win,
                                              long long s, long long b, long long d, BlockShared &sh,
                                              unsigned chk_mask) {
    constexpr bool CHK = PACK;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    unsigned bad = 0;
    // after a checked fill: restart with split bins if any add left the range
    auto overflowed = [&]() -> bool {
        if constexpr (CHK) {
            if (__syncthreads_or(bad & chk_mask)) {
                if (threadIdx.x == 0) atomicAdd(a.ticket + 3, 1u);  // eucalc_k2_restarts
                for (int i = threadIdx.x; i < win; i += kBlockThreads) hist[i] = 0;
                __syncthreads();
                return true;
            }
            return false;
        } else {
            __syncthreads();
            return false;
        }
    };
    Hist<PACK, true> hs;
    hs.c = hist;
    hs.j = hist + win;
    hs.nb = win;
    const RecT *recs = reinterpret_cast<const RecT *>(a.rec);
    const DirInfo di = a.dirs[d];
    const RecT *list = recs + (b * a.Q + di.q) * a.vcap;
    const int32_t *toff = a.tile_off + (b * a.Q + di.q) * (long long)(a.ntiles + 1);
    const int n = a.count[b * a.Q + di.q];
    const int nwin = (di.R + win - 1) / win;
    const bool cull = nwin > 1 && a.ntiles > 1;
    // each warp owns a contiguous, 128-aligned range of the window
    const int per = ((win / kBlockWarps) + kGroup - 1) / kGroup * kGroup;
    // phase A: counts over all windows
    long long nc = 0, no = 0;
    for (int w = 0; w < nwin; ++w) {
        const int lo = w * win, wb = min(win, di.R - lo);
        fill_window<DP, CHK>(a, list, toff, n, di, lo, wb, cull, hs, sh.hit, &sh.nhit, bad, chk_mask != 0);
        if (overflowed()) return false;
        int c = 0, o = 0;
        const int b0 = min(wb, warp * per), b1 = min(wb, b0 + per);
        for (int base = b0; base < b1; base += kGroup) count_group(hs, base, c, o, nwin > 1);
        c = warp_sum(c);
        o = warp_sum(o);
        if (lane == 0) {
            sh.wsum[warp][0] = c;
            sh.wsum[warp][1] = o;
        }
        __syncthreads();
        for (int k = 0; k < kBlockWarps; ++k) {
            nc += sh.wsum[k][0];
            no += sh.wsum[k][1];
        }
        __syncthreads();
    }
    if (warp == 0) {
        long long ec, eo;
        seg_lookback(a.flags, s, nc, no, ec, eo);
        if (lane == 0) {
            sh.exc[0] = ec;
            sh.exc[1] = eo;
            write_offsets(a, s, ec, eo, nc, no);
        }
    }
    __syncthreads();
    // phase B: emit window by window
    long long pc_carry = sh.exc[0], po_carry = sh.exc[1];
    int e_carry = 0, r_carry = 0;
    double ht = 0.0;
    const long long ht_off = outp.tab ? ht_tab_off(a, di) : 0;
    for (int w = 0; w < nwin; ++w) {
        const int lo = w * win, wb = min(win, di.R - lo);
        if (nwin > 1) {
            // unchecked: phase A's checks proved every bin's final sums in range, and
            // packed sums are exact for in-range finals whatever the add order
            fill_window<DP, false>(a, list, toff, n, di, lo, wb, cull, hs, sh.hit, &sh.nhit, bad, false);
            __syncthreads();
        }
        const int b0 = min(wb, warp * per), b1 = min(wb, b0 + per);
        int c = 0, o = 0, sc = 0, sj = 0;
        for (int base = b0; base < b1; base += kGroup) {
            int wc[4], wj[4];
            hs.load4(base + 4 * lane, wc, wj, false);
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                c += wc[q] != 0;
                o += wj[q] != 0;
                sc += wc[q];
                sj += wj[q];
            }
        }
        c = warp_sum(c);
        o = warp_sum(o);
        sc = warp_sum(sc);
        sj = warp_sum(sj);
        if (lane == 0) {
            sh.wsum[warp][0] = c;
            sh.wsum[warp][1] = o;
            sh.wsum[warp][2] = sc;
            sh.wsum[warp][3] = sj;
        }
        __syncthreads();
        int pc = (int)pc_carry, po = (int)po_carry;
        int er = e_carry, rr = r_carry;
        long long tc = 0, to = 0;
        int tsc = 0, tsj = 0;
        for (int k = 0; k < kBlockWarps; ++k) {
            if (k < warp) {
                pc += sh.wsum[k][0];
                po += sh.wsum[k][1];
                er += sh.wsum[k][2];
                rr += sh.wsum[k][3];
            }
            tc += sh.wsum[k][0];
            to += sh.wsum[k][1];
            tsc += sh.wsum[k][2];
            tsj += sh.wsum[k][3];
        }
        for (int base = b0; base < b1; base += kGroup)
            emit_group<kModeAny>(outp, hs, base, di.hlo + lo, er, rr, pc, po, ht, ht_off);
        pc_carry += tc;
        po_carry += to;
        e_carry += tsc;
        r_carry += tsj;
        __syncthreads();
    }
    if (outp.tab) {  // fused HT: warp partials, then a fixed-order sum over warps
        for (int k = 16; k; k >>= 1) ht += __shfl_xor_sync(0xffffffffu, ht, k);
        if (lane == 0) sh.ht[warp] = ht;
        __syncthreads();
        if (threadIdx.x == 0) {
            double t = 0.0;
            for (int k = 0; k < kBlockWarps; ++k) t += sh.ht[k];
            ht_write(a, s, t);
        }
    }
    return true;
}

// Staged variant (the pipelined block kernel): ONE fill per window, the
// segment's entries go to the staging buffer `base` at segment-local positions;
// its counts end in sh.cnt (nc, no) and its HT (if fused) is written. Nothing is
// published. Returns false when a checked packed fill flagged (rerun split).
template <bool PACK, int DP, typename RecT, typename OutT, typename SH = BlockShared>
__device__ __forceinline__ bool block_segment_staged(const K2Args &a, const OutPtrs<OutT> &outp, unsigned *hist,
                                                     int win, long long s, long long b, long long d,
                                                     SH &sh, unsigned chk_mask, OutT *base) {
    constexpr bool CHK = PACK;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    unsigned bad = 0;
    auto overflowed = [&]() -> bool {
        if constexpr (CHK) {
            if (__syncthreads_or(bad & chk_mask)) {
                if (threadIdx.x == 0) atomicAdd(a.ticket + 3, 1u);  // eucalc_k2_restarts
                for (int i = threadIdx.x; i < win; i += kBlockThreads) hist[i] = 0;
                __syncthreads();
                return true;
            }
            return false;
        } else {
            __syncthreads();
            return false;
        }
    };
    Hist<PACK, true> hs;
    hs.c = hist;
    hs.j = hist + win;
    const RecT *recs = reinterpret_cast<const RecT *>(a.rec);
    const DirInfo di = a.dirs[d];
    const RecT *list = recs + (b * a.Q + di.q) * a.vcap;
    const int32_t *toff = a.tile_off + (b * a.Q + di.q) * (long long)(a.ntiles + 1);
    const int n = a.count[b * a.Q + di.q];
    const int nwin = (di.R + win - 1) / win;
    const bool cull = nwin > 1 && a.ntiles > 1;
    const int per = ((win / kBlockWarps) + kGroup - 1) / kGroup * kGroup;
    OutPtrs<OutT> scr = outp;
    scr.eh = base;
    scr.ev = base + a.stage_cap;
    scr.cv = base + 2 * a.stage_cap;
    scr.ch = base + 3 * a.stage_cap;
    scr.oh = base + 4 * a.stage_cap;
    scr.ov = base + 5 * a.stage_cap;
    scr.ect = outp.ect || outp.cls;  // staged heights serve both (T_c = T)
    scr.alias = true;
    scr.cap = (a.units || a.stage_base) ? di.R : a.stage_cap;  // the segment's slot; else the CTA's buffer
    hs.nb = win;
    int pc_carry = 0, po_carry = 0, e_carry = 0, r_carry = 0;
    double ht = 0.0;
    const long long ht_off = outp.tab ? ht_tab_off(a, di) : 0;
    for (int w = 0; w < nwin; ++w) {
        const int lo = w * win, wb = min(win, di.R - lo);
        fill_window<DP, CHK>(a, list, toff, n, di, lo, wb, cull, hs, sh.hit, &sh.nhit, bad, chk_mask != 0);
        if (overflowed()) return false;
        const int b0 = min(wb, warp * per), b1 = min(wb, b0 + per);
        int c = 0, o = 0, sc = 0, sj = 0;
        for (int base = b0; base < b1; base += kGroup) {
            int wc[4], wj[4];
            hs.load4(base + 4 * lane, wc, wj, false);
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                c += wc[q] != 0;
                o += wj[q] != 0;
                sc += wc[q];
                sj += wj[q];
            }
        }
        c = warp_sum(c);
        o = warp_sum(o);
        sc = warp_sum(sc);
        sj = warp_sum(sj);
        if (lane == 0) {
            sh.wsum[warp][0] = c;
            sh.wsum[warp][1] = o;
            sh.wsum[warp][2] = sc;
            sh.wsum[warp][3] = sj;
        }
        __syncthreads();
        int pc = pc_carry, po = po_carry, er = e_carry, rr = r_carry;
        int tc = 0, to = 0, tsc = 0, tsj = 0;
        for (int k = 0; k < kBlockWarps; ++k) {
            if (k < warp) {
                pc += sh.wsum[k][0];
                po += sh.wsum[k][1];
                er += sh.wsum[k][2];
                rr += sh.wsum[k][3];
            }
            tc += sh.wsum[k][0];
            to += sh.wsum[k][1];
            tsc += sh.wsum[k][2];
            tsj += sh.wsum[k][3];
        }
        for (int base = b0; base < b1; base += kGroup)
            emit_group<kModeAny>(scr, hs, base, di.hlo + lo, er, rr, pc, po, ht, ht_off);
        pc_carry += tc;
        po_carry += to;
        e_carry += tsc;
        r_carry += tsj;
        __syncthreads();
    }
    if (outp.tab) {  // fused HT: warp partials, then a fixed-order sum over warps
        for (int k = 16; k; k >>= 1) ht += __shfl_xor_sync(0xffffffffu, ht, k);
        if (lane == 0) sh.ht[warp] = ht;
        __syncthreads();
        if (threadIdx.x == 0) {
            double t = 0.0;
            for (int k = 0; k < kBlockWarps; ++k) t += sh.ht[k];
            ht_write(a, s, t);
        }
    }
    if (threadIdx.x == 0) {
        sh.cnt[0] = pc_carry;
        sh.cnt[1] = po_carry;
    }
    return true;
}

// Staged entries of a resolved segment -> the CSR (four loads in flight per thread).
template <typename OutT>
__device__ __forceinline__ void copy_out(const OutPtrs<OutT> &outp, const OutT *base, long long cap, long long ec,
                                         long long eo, int nc, int no) {
    const OutT *eh = base, *ev = base + cap, *cv = base + 2 * cap, *ch = base + 3 * cap, *oh = base + 4 * cap,
               *ov = base + 5 * cap;
    EU_DCHECK(nc <= cap && no <= cap && ec + nc <= outp.cap && eo + no <= outp.cap);
    constexpr int U = 4;
    if (outp.ect || outp.cls) {
        for (int i0 = threadIdx.x; i0 < nc; i0 += U * kBlockThreads) {
            OutT h[U], v[U], c[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int i = i0 + u * kBlockThreads;
                if (i < nc) {
                    h[u] = __ldcs(eh + i);
                    v[u] = __ldcs(ev + i);
                    c[u] = __ldcs(cv + i);
                }
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int i = i0 + u * kBlockThreads;
                if (i < nc) {
                    if (outp.ect) {
                        __stcs(outp.eh + ec + i, h[u]);
                        __stcs(outp.ev + ec + i, v[u]);
                    }
                    if (outp.cls) {
                        if (!outp.alias) __stcs(outp.ch + ec + i, h[u]);
                        __stcs(outp.cv + ec + i, c[u]);
                    }
                }
            }
        }
    }
    if (outp.ord) {
        for (int i0 = threadIdx.x; i0 < no; i0 += U * kBlockThreads) {
            OutT h[U], v[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int i = i0 + u * kBlockThreads;
                if (i < no) {
                    h[u] = __ldcs(oh + i);
                    v[u] = __ldcs(ov + i);
                }
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int i = i0 + u * kBlockThreads;
                if (i < no) {
                    __stcs(outp.oh + eo + i, h[u]);
                    __stcs(outp.ov + eo + i, v[u]);
                }
            }
        }
    }
    (void)ch;
}

// Block regime. A segment uses packed 16+16 bins (one atomic per record, windows
// of 2*win bins) when its bins provably stay below 2^15: every bin holds at most
// di.line records (the vertices of one height level) of |a|+|b| <= max_rec, and
// no more than the list's sum |a|+|b|; else split bins (two int32 arrays, windows
// of win bins). `hist` is cleared on entry and left cleared by every segment.
template <typename RecT, typename OutT, int DP>
__global__ void __launch_bounds__(kBlockThreads, 1) k2_block(K2Args a, long long nseg, int win) {
    extern __shared__ __align__(16) unsigned hist[];
    __shared__ BlockShared sh;
    const OutPtrs<OutT> outp(a);
    for (int i = threadIdx.x; i < 2 * win; i += kBlockThreads) hist[i] = 0;
    // packed bins: proven exact (no check), or checked (rerun split on a flag)
    auto packed_mask = [&](long long d, bool &use_packed) -> unsigned {
        const long long bin_bound = min((long long)a.dirs[d].line * (long long)a.max_rec, (long long)a.max_abs_sum);
        const bool proven = bin_bound < 32768;
        use_packed = proven || (a.max_rec < 16384 && !a.no_chk);
        return proven ? 0u : a.chk_mask;
    };
    if (a.stage && a.stage_base) {
        // Slot mode: every segment is filled once and emitted into its own fixed staging
        // slot (R_d entries per array, as in the unit path), its counts go to cnt_c/cnt_o;
        // k2_scan then turns the counts into the CSR offsets and k2_unit_copy moves the
        // staged entries there at copy-kernel bandwidth - no look-back between segments
        // and no copy-out inside this kernel's segment loop.
        OutT *stage = reinterpret_cast<OutT *>(a.stage);
        while (true) {
            __syncthreads();
            if (threadIdx.x == 0) sh.seg = (long long)atomicAdd(a.ticket, 1u);
            __syncthreads();
            const long long t = sh.seg;
            if (t >= nseg) break;
            // any order is valid here: the directions with the largest height range first, so
            // the last wave holds the shortest segments
            const long long b = t / a.D, d = a.seg_order ? a.seg_order[t % a.D] : t % a.D, s = b * a.D + d;
            OutT *slot = stage + b * a.stage_img + a.stage_base[d];
            bool packed;
            const unsigned m = packed_mask(d, packed);
            if (!packed || !block_segment_staged<true, DP, RecT, OutT>(a, outp, hist, 2 * win, s, b, d, sh, m, slot))
                block_segment_staged<false, DP, RecT, OutT>(a, outp, hist, win, s, b, d, sh, 0u, slot);
            __syncthreads();
            if (threadIdx.x == 0) {
                a.cnt_c[s] = sh.cnt[0];
                a.cnt_o[s] = sh.cnt[1];
            }
        }
        return;
    }
    if (a.stage) {
        // Pipelined: segment s is filled and emitted into staging buffer `cur` and
        // its aggregate published; then the PREVIOUS segment of this CTA is looked
        // back (its predecessors have had a whole segment's time to publish) and
        // copied from the other buffer to the CSR.
        int cur = 0;
        long long prev = -1;
        int pnc = 0, pno = 0;
        OutT *stage = reinterpret_cast<OutT *>(a.stage);
        while (true) {
            __syncthreads();
            if (threadIdx.x == 0) sh.seg = (long long)atomicAdd(a.ticket, 1u);
            __syncthreads();
            const long long s = sh.seg;
            int nc = 0, no = 0;
            if (s < nseg) {
                const long long b = s / a.D, d = s % a.D;
                OutT *buf = stage + ((long long)blockIdx.x * 2 + cur) * 6 * a.stage_cap;
                bool packed;
                const unsigned m = packed_mask(d, packed);
                if (!packed || !block_segment_staged<true, DP, RecT, OutT>(a, outp, hist, 2 * win, s, b, d, sh, m, buf))
                    block_segment_staged<false, DP, RecT, OutT>(a, outp, hist, win, s, b, d, sh, 0u, buf);
                __syncthreads();
                nc = sh.cnt[0];
                no = sh.cnt[1];
                if (threadIdx.x == 0) seg_publish(a.flags, s, nc, no);
            }
            if (prev >= 0) {
                if (threadIdx.x < 32) {
                    long long ec, eo;
                    seg_lookback<true>(a.flags, prev, pnc, pno, ec, eo);
                    if (threadIdx.x == 0) {
                        sh.exc[0] = ec;
                        sh.exc[1] = eo;
                        write_offsets(a, prev, ec, eo, pnc, pno);
                    }
                }
                __syncthreads();
                const OutT *pbuf = stage + ((long long)blockIdx.x * 2 + (cur ^ 1)) * 6 * a.stage_cap;
                copy_out(outp, pbuf, a.stage_cap, sh.exc[0], sh.exc[1], pnc, pno);
            }
            if (s >= nseg) break;
            prev = s;
            pnc = nc;
            pno = no;
            cur ^= 1;
        }
        return;
    }
    while (true) {
        __syncthreads();
        if (threadIdx.x == 0) sh.seg = (long long)atomicAdd(a.ticket, 1u);
        __syncthreads();
        const long long s = sh.seg;
        if (s >= nseg) break;
        const long long b = s / a.D, d = s % a.D;
        bool packed;
        const unsigned m = packed_mask(d, packed);
        if (!packed || !block_segment<true, DP, RecT, OutT>(a, outp, hist, 2 * win, s, b, d, sh, m))
            block_segment<false, DP, RecT, OutT>(a, outp, hist, win, s, b, d, sh, 0u);
    }
}

// ----------------------------------------------------------------------------- unit kernel
// Block regime with several directions per pass over a list ("units"): the
// directions of one image that read the same pair list from the same side
// (same orthant, Lemma 3) are grouped into units of G <= kUnitMax whose
// packed histograms fit shared memory together (sum of their 128-padded R).
// A CTA streams the list ONCE per unit and adds every record into the G
// histograms (one dp4a + one shared atomic per record and direction), so the
// record loads, the weight-word extraction and the loop overhead are shared by
// G directions. Each histogram is then emitted (the paper's cumulative sums,
// P:126-128) into the segment's fixed staging slot (capacity R_d entries per
// stream), its counts go to cnt_c/cnt_o; k2_scan turns the counts into the CSR
// offsets and k2_unit_copy moves the staged entries there. Units are taken by
// ticket in any order (no look-back between segments).
// Packed bins are checked exactly as in k2_block (Hist::add_chk) unless a bound
// proves them for every direction of the unit; a flagged unit is redone one
// direction at a time with split bins (block_segment_staged, one window).
constexpr int kUnitMax = 4;
// the unit kernel's shared state (no culled-tile list: its segments are single-window)
struct UnitShared {
    long long seg;
    int cnt[2];
    int wsum[kBlockWarps][4];
    double ht[kBlockWarps];
    int hit[1];
    int nhit;
};
constexpr size_t kUnitSmem = 222 * 1024;                // dynamic: 227 KB per CTA minus UnitShared
constexpr int kUnitWords = (int)(kUnitSmem / 4);  // packed words of shared histogram per CTA


// Per-unit parameters of the fill: per direction the packed int8 direction, -hlo
// and the shared byte address of its histogram.
struct UnitParams {
    int xs8[kUnitMax], nhlo[kUnitMax];
    unsigned sb[kUnitMax];
    int nb[kUnitMax];  // R of each direction (device checks)
};

// Adds records threadIdx.x + k * kBlockThreads of `list` into the G packed
// histograms: per record one weight word, per record and direction one dp4a
// (height - hlo), the bank swizzle and one shared atomic (checked: the returned
// word biased and OR-ed into `bad`). The parameters are copied to registers once.
template <bool CHK, bool SWAP, int G>
__device__ __forceinline__ unsigned unit_fill(const uint2 *list, int n, const UnitParams &pp, unsigned bias) {
    constexpr int U = 4;
    constexpr int step = kBlockThreads;
    int xs8[G], nhlo[G];
    unsigned sb[G];
#pragma unroll
    for (int g = 0; g < G; ++g) {
        xs8[g] = pp.xs8[g];
        nhlo[g] = pp.nhlo[g];
        sb[g] = pp.sb[g];
    }
    unsigned bad = 0;
    auto one = [&](const uint2 r) {
        const unsigned w = packed_word<SWAP>(r.y);
#pragma unroll
        for (int g = 0; g < G; ++g) {
            int h;
            asm("dp4a.u32.s32 %0, %1, %2, %3;" : "=r"(h) : "r"(r.x), "r"(xs8[g]), "r"(nhlo[g]));
            EU_DCHECK(h >= 0 && h < pp.nb[g]);
            const unsigned addr = sb[g] + ((unsigned)swz(h) << 2);
            if constexpr (CHK) bad |= atom_smem(addr, w) + w + bias;
            else red_smem(addr, w);
        }
    };
    int i = threadIdx.x;
    for (; i + (U - 1) * step < n; i += U * step) {
        uint2 r[U];
#pragma unroll
        for (int u = 0; u < U; ++u) r[u] = __ldg(list + i + u * step);
#pragma unroll
        for (int u = 0; u < U; ++u) one(r[u]);
    }
    for (; i < n; i += step) one(__ldg(list + i));
    return bad;
}

template <bool CHK, bool SWAP>
__device__ __noinline__ unsigned unit_fill_any(const uint2 *list, int n, int G, UnitParams pp, unsigned bias) {
    switch (G) {
    case 1: return unit_fill<CHK, SWAP, 1>(list, n, pp, bias);
    case 2: return unit_fill<CHK, SWAP, 2>(list, n, pp, bias);
    case 3: return unit_fill<CHK, SWAP, 3>(list, n, pp, bias);
    default: return unit_fill<CHK, SWAP, 4>(list, n, pp, bias);
    }
}

// Emits one packed histogram (R bins at hist, single window) of segment s into
// its staging slot `base` (arrays at stride cap); counts -> sh.cnt, HT written.
template <typename OutT>
__device__ __noinline__ void unit_emit(const K2Args &a, const OutPtrs<OutT> &outp, unsigned *hist, int R,
                                          long long s, const DirInfo &di, UnitShared &sh, OutT *base,
                                          long long cap) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    Hist<true, true> hs;
    hs.c = hist;
    hs.j = hist;
    hs.nb = R;
    OutPtrs<OutT> scr = outp;
    scr.cap = R;  // the segment's staging slot
    scr.eh = base;
    scr.ev = base + cap;
    scr.cv = base + 2 * cap;
    scr.ch = base + 3 * cap;
    scr.oh = base + 4 * cap;
    scr.ov = base + 5 * cap;
    scr.ect = outp.ect || outp.cls;  // staged heights serve both (T_c = T)
    scr.alias = true;
    const int per = ((R + kBlockWarps - 1) / kBlockWarps + kGroup - 1) / kGroup * kGroup;
    const int b0 = min(R, warp * per), b1 = min(R, b0 + per);
    int c = 0, o = 0, sc = 0, sj = 0;
    for (int bb = b0; bb < b1; bb += kGroup) {
        int wc[4], wj[4];
        hs.load4(bb + 4 * lane, wc, wj, false);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            c += wc[q] != 0;
            o += wj[q] != 0;
            sc += wc[q];
            sj += wj[q];
        }
    }
    c = warp_sum(c);
    o = warp_sum(o);
    sc = warp_sum(sc);
    sj = warp_sum(sj);
    if (lane == 0) {
        sh.wsum[warp][0] = c;
        sh.wsum[warp][1] = o;
        sh.wsum[warp][2] = sc;
        sh.wsum[warp][3] = sj;
    }
    __syncthreads();
    int pc = 0, po = 0, er = 0, rr = 0, tc = 0, to = 0;
    for (int k = 0; k < kBlockWarps; ++k) {
        if (k < warp) {
            pc += sh.wsum[k][0];
            po += sh.wsum[k][1];
            er += sh.wsum[k][2];
            rr += sh.wsum[k][3];
        }
        tc += sh.wsum[k][0];
        to += sh.wsum[k][1];
    }
    double ht = 0.0;
    const long long ht_off = outp.tab ? ht_tab_off(a, di) : 0;
    for (int bb = b0; bb < b1; bb += kGroup) emit_group<kModeAny>(scr, hs, bb, di.hlo, er, rr, pc, po, ht, ht_off);
    if (outp.tab) {  // fused HT: warp partials, then a fixed-order sum over warps
        for (int k = 16; k; k >>= 1) ht += __shfl_xor_sync(0xffffffffu, ht, k);
        if (lane == 0) sh.ht[warp] = ht;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        if (outp.tab) {
            double t = 0.0;
            for (int k = 0; k < kBlockWarps; ++k) t += sh.ht[k];
            ht_write(a, s, t);
        }
        a.cnt_c[s] = tc;
        a.cnt_o[s] = to;
    }
}

template <typename OutT>
__device__ __noinline__ void unit_split_segment(const K2Args &a, const OutPtrs<OutT> &outp, unsigned *hist,
                                                int split_win, long long s, long long b, long long d,
                                                UnitShared &sh, OutT *base) {
    block_segment_staged<false, 3, Rec16, OutT, UnitShared>(a, outp, hist, split_win, s, b, d, sh, 0u, base);
    __syncthreads();
    if (threadIdx.x == 0) {
        a.cnt_c[s] = sh.cnt[0];
        a.cnt_o[s] = sh.cnt[1];
    }
}

template <typename OutT>
__global__ void __launch_bounds__(kBlockThreads, 1) k2_unit(K2Args a, int split_win) {
    extern __shared__ __align__(16) unsigned hist[];
    __shared__ UnitShared sh;
    const OutPtrs<OutT> outp(a);
    OutT *stage = reinterpret_cast<OutT *>(a.stage);
    const unsigned hist_sa = (unsigned)__cvta_generic_to_shared(hist);
    for (int i = threadIdx.x; i < kUnitWords; i += kBlockThreads) hist[i] = 0;
    const long long total = a.nunits * a.batch;
    while (true) {
        __syncthreads();
        if (threadIdx.x == 0) sh.seg = (long long)atomicAdd(a.ticket, 1u);
        __syncthreads();
        const long long t = sh.seg;
        if (t >= total) break;
        // image-major, heaviest image first: the CTAs in flight stream the same few lists
        // (L2) and the short units of light images fill the tail of the heavy ones;
        // without an order, images interleaved (equal units of all images run together)
        const long long b = a.img_order ? a.img_order[t / a.nunits] : t % a.batch;
        const int4 un = a.units[a.img_order ? t % a.nunits : t / a.batch];  // {first index into unit_dirs, G, q, swap}
        const int G = un.y;
        UnitParams pp;
        int base[kUnitMax];
        bool proven = true;
        int off = 0;
#pragma unroll
        for (int g = 0; g < kUnitMax; ++g) {
            pp.xs8[g] = 0;
            pp.nhlo[g] = 0;
            pp.nb[g] = 0;
            base[g] = 0;
            if (g < G) {
                const DirInfo &di = a.dirs[a.unit_dirs[un.x + g]];
                pp.xs8[g] = di.xs8;
                pp.nhlo[g] = -di.hlo;
                pp.nb[g] = di.R;
                base[g] = off;
                off += (di.R + kGroup - 1) / kGroup * kGroup;
                proven = proven && min((long long)di.line * a.max_rec, (long long)a.max_abs_sum) < 32768;
            }
            pp.sb[g] = hist_sa + 4u * (unsigned)base[g];
        }
        const uint2 *list = reinterpret_cast<const uint2 *>(a.rec) + (b * a.Q + un.z) * a.vcap;
        const int n = a.count[b * a.Q + un.z];
        unsigned bad;
        if (proven) bad = un.w ? unit_fill_any<false, true>(list, n, G, pp, 0u) : unit_fill_any<false, false>(list, n, G, pp, 0u);
        else bad = un.w ? unit_fill_any<true, true>(list, n, G, pp, a.chk_bias) : unit_fill_any<true, false>(list, n, G, pp, a.chk_bias);
        if (__syncthreads_or(proven ? 0u : (bad & a.chk_mask))) {
            // a packed bin left the checked range: redo each direction with split bins
            if (threadIdx.x == 0) atomicAdd(a.ticket + 3, (unsigned)G);  // eucalc_k2_restarts: per segment
            for (int i = threadIdx.x; i < kUnitWords; i += kBlockThreads) hist[i] = 0;
            __syncthreads();
            for (int g = 0; g < G; ++g) {
                const long long d = a.unit_dirs[un.x + g], s = b * a.D + d;
                unit_split_segment<OutT>(a, outp, hist, split_win, s, b, d, sh,
                                         stage + b * a.stage_img + a.stage_base[d]);
            }
            continue;
        }
        for (int g = 0; g < G; ++g) {
            const long long d = a.unit_dirs[un.x + g], s = b * a.D + d;
            const DirInfo di = a.dirs[d];
            unit_emit<OutT>(a, outp, hist + base[g], di.R, s, di, sh, stage + b * a.stage_img + a.stage_base[d],
                            a.stage_cap);
        }
    }
}

// Staged entries of every segment -> the CSR (one CTA per segment, grid-stride;
// eight elements per array in flight per thread before their stores).
template <typename OutT>
__global__ void __launch_bounds__(512) k2_unit_copy(K2Args a) {
    constexpr int U = 8;
    const OutPtrs<OutT> outp(a);
    const OutT *stage = reinterpret_cast<const OutT *>(a.stage);
    const long long S = a.batch * a.D, cap = a.stage_cap;
    const int T = blockDim.x;
    for (long long s = blockIdx.x; s < S; s += gridDim.x) {
        const long long b = s / a.D, d = s - b * a.D;
        const OutT *bs = stage + b * a.stage_img + a.stage_base[d];
        const int nc = a.cnt_c[s], no = a.cnt_o[s];
        const long long ec = a.do_ect ? a.ect.off[s] : a.do_cls ? a.cls.off[s] : 0;
        const long long eo = a.do_ord ? a.ord.off[s] : 0;
        EU_DCHECK(nc <= a.dirs[d].R && no <= a.dirs[d].R && ec + nc <= outp.cap && eo + no <= outp.cap);
        if (outp.ect || outp.cls) {
            for (int i0 = threadIdx.x; i0 < nc; i0 += U * T) {
                OutT h[U], v[U], c[U];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int i = i0 + u * T;
                    if (i < nc) {
                        h[u] = bs[i];
                        v[u] = bs[cap + i];
                        c[u] = bs[2 * cap + i];
                    }
                }
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int i = i0 + u * T;
                    if (i < nc) {
                        if (outp.ect) {
                            outp.eh[ec + i] = h[u];
                            outp.ev[ec + i] = v[u];
                        }
                        if (outp.cls) {
                            if (!outp.alias) outp.ch[ec + i] = h[u];
                            outp.cv[ec + i] = c[u];
                        }
                    }
                }
            }
        }
        if (outp.ord) {
            for (int i0 = threadIdx.x; i0 < no; i0 += U * T) {
                OutT h[U], v[U];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int i = i0 + u * T;
                    if (i < no) {
                        h[u] = bs[4 * cap + i];
                        v[u] = bs[5 * cap + i];
                    }
                }
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int i = i0 + u * T;
                    if (i < no) {
                        outp.oh[eo + i] = h[u];
                        outp.ov[eo + i] = v[u];
                    }
                }
            }
        }
    }
}

template <typename OutT>
cudaError_t launch_unit_t(const K2Args &a, cudaStream_t s, int num_sms) {
    auto kern = k2_unit<OutT>;
    cudaError_t e = prepare_kernel((const void *)kern, kBlockThreads, kUnitSmem, nullptr);
    if (e != cudaSuccess) return e;
    const long long total = a.nunits * a.batch, S = a.batch * a.D;
    if (total == 0) return cudaSuccess;
    const int split_win = (int)(kBlockSmem / 8) / kGroup * kGroup;
    kern<<<(unsigned)std::min<long long>(total, num_sms), kBlockThreads, kUnitSmem, s>>>(a, split_win);
    const long long ntiles = (S + 1 + kScanTile - 1) / kScanTile;
    k2_scan<<<(unsigned)ntiles, kScanThreads, 0, s>>>(a, a.cnt_c, a.cnt_o, S, a.flags);
    k2_unit_copy<OutT><<<(unsigned)std::min<long long>(S, 4LL * num_sms), 512, 0, s>>>(a);
    count_launch(3);
    return cudaGetLastError();
}

template <typename RecT, typename OutT, bool PACK>
cudaError_t launch_t(const K2Args &a, cudaStream_t s, int num_sms) {
    const long long nseg = a.batch * a.D;
    constexpr int words = PACK ? 1 : 2;
    // warp regime: whole histogram per warp, small lists
    const int rcap = (a.R_max + kGroup - 1) / kGroup * kGroup;
    const size_t per_warp = (size_t)rcap * 4 * words;
    int warps = (int)std::min<size_t>(8, (200 * 1024) / per_warp);
    if (warps >= 2 && a.max_count <= 32768) {
        const int threads = warps * 32;
        const size_t smem = per_warp * warps;
        auto kc = k2w_count<RecT, PACK>;
        void (*ke)(K2Args, int) = k2w_emit<RecT, OutT, PACK, kModeAny>;
        if (std::is_same<RecT, Rec16>::value) {
            const int mode = (a.do_ect ? kEct : 0) | (a.do_ord ? kOrd : 0) | (a.do_cls ? kCls : 0) |
                             (a.do_cls && a.cls_alias ? kAlias : 0) | (a.ht_tab ? kHt : 0);
            switch (mode) {
            case kEct: ke = k2w_emit<RecT, OutT, PACK, kEct>; break;
            case kOrd | kCls: ke = k2w_emit<RecT, OutT, PACK, kOrd | kCls>; break;
            case kEct | kOrd | kCls: ke = k2w_emit<RecT, OutT, PACK, kEct | kOrd | kCls>; break;
            case kEct | kOrd | kCls | kAlias: ke = k2w_emit<RecT, OutT, PACK, kEct | kOrd | kCls | kAlias>; break;
            case kEct | kOrd | kCls | kAlias | kHt:
                ke = k2w_emit<RecT, OutT, PACK, kEct | kOrd | kCls | kAlias | kHt>;
                break;
            default: break;
            }
        }
        int occ = 0, occ2 = 0;
        cudaError_t e = prepare_kernel((const void *)kc, threads, smem, &occ);
        if (e == cudaSuccess) e = prepare_kernel((const void *)ke, threads, smem, &occ2);
        if (e != cudaSuccess) return e;
        const long long wblocks = (nseg + warps - 1) / warps;
        const long long grid = std::min<long long>(wblocks, (long long)std::max(occ, 1) * num_sms);
        kc<<<(unsigned)grid, threads, smem, s>>>(a, rcap, a.cnt_c, a.cnt_o);
        const long long ntiles = (nseg + 1 + kScanTile - 1) / kScanTile;
        k2_scan<<<(unsigned)ntiles, kScanThreads, 0, s>>>(a, a.cnt_c, a.cnt_o, nseg, a.flags);
        const long long grid2 = std::min<long long>(wblocks, (long long)std::max(occ2, 1) * num_sms);
        ke<<<(unsigned)grid2, threads, smem, s>>>(a, rcap);
        count_launch(3);
        return cudaGetLastError();
    }
    const int win = (int)(kBlockSmem / 8) / kGroup * kGroup;  // split bins; packed segments use 2 * win
    auto kern = a.dp == 3 ? k2_block<RecT, OutT, 3> : a.dp == 2 ? k2_block<RecT, OutT, 2> : k2_block<RecT, OutT, 0>;
    cudaError_t e = prepare_kernel((const void *)kern, kBlockThreads, kBlockSmem, nullptr);
    if (e != cudaSuccess) return e;
    long long grid = std::min<long long>(nseg, num_sms);
    kern<<<(unsigned)grid, kBlockThreads, kBlockSmem, s>>>(a, nseg, win);
    count_launch();
    if (a.stage && a.stage_base) {  // slot mode: offsets from the counts, then the staged entries to the CSR
        const long long ntiles = (nseg + 1 + kScanTile - 1) / kScanTile;
        k2_scan<<<(unsigned)ntiles, kScanThreads, 0, s>>>(a, a.cnt_c, a.cnt_o, nseg, a.flags);
        k2_unit_copy<OutT><<<(unsigned)std::min<long long>(nseg, 8LL * num_sms), 512, 0, s>>>(a);
        count_launch(2);
    }
    return cudaGetLastError();
}

template <typename RecT, typename OutT>
cudaError_t launch_p(const K2Args &a, cudaStream_t s, int num_sms) {
    return a.pack16 ? launch_t<RecT, OutT, true>(a, s, num_sms) : launch_t<RecT, OutT, false>(a, s, num_sms);
}
template <typename RecT>
cudaError_t launch_o(const K2Args &a, cudaStream_t s, int num_sms) {
#ifdef EUCALC_DEV_FAST  // development builds (libeucalc_dev.so): only 32-bit outputs are instantiated
    return a.elem_bytes == 4 ? launch_p<RecT, int32_t>(a, s, num_sms) : cudaErrorNotSupported;
#else
    switch (a.elem_bytes) {
    case 2: return launch_p<RecT, int16_t>(a, s, num_sms);
    case 4: return launch_p<RecT, int32_t>(a, s, num_sms);
    default: return launch_p<RecT, int64_t>(a, s, num_sms);
    }
#endif
}

}  // namespace

cudaError_t launch_csr_scan(const K2Args &a, const int *cnt_c, const int *cnt_o, long long S, cudaStream_t s) {
    const long long ntiles = (S + 1 + kScanTile - 1) / kScanTile;
    k2_scan<<<(unsigned)ntiles, kScanThreads, 0, s>>>(a, cnt_c, cnt_o, S, a.flags);
    count_launch();
    return cudaGetLastError();
}

size_t k2_stage_bytes(const K2Args &a, int num_sms, int64_t *cap) {
    *cap = 0;
    const long long nseg = a.batch * a.D;
    const int words = a.pack16 ? 1 : 2;
    const int rcap = (a.R_max + kGroup - 1) / kGroup * kGroup;
    const size_t per_warp = (size_t)rcap * 4 * words;
    const int warps = (int)std::min<size_t>(8, (200 * 1024) / per_warp);
    if (nseg == 0 || (warps >= 2 && a.max_count <= 32768)) return 0;  // warp regime
    // per stream and segment: at most min(list length, R) entries
    const int64_t c = std::max<int64_t>(1, std::min<int64_t>(a.max_count, a.R_max));
    const long long grid = std::min<long long>(nseg, num_sms);
    const size_t bytes = (size_t)grid * 2 * 6 * (size_t)c * (size_t)a.elem_bytes;  // two buffers per CTA
    if (bytes > (size_t(4) << 30)) return 0;
    *cap = c;
    return bytes;
}

cudaError_t launch_k2(const K2Args &a, cudaStream_t s, int num_sms) {
#ifdef EUCALC_DEV_FAST
    if (a.units) return a.elem_bytes == 4 ? launch_unit_t<int32_t>(a, s, num_sms) : cudaErrorNotSupported;
    return a.wide ? cudaErrorNotSupported : launch_o<Rec16>(a, s, num_sms);
#else
    if (a.units) {
        switch (a.elem_bytes) {
        case 2: return launch_unit_t<int16_t>(a, s, num_sms);
        case 4: return launch_unit_t<int32_t>(a, s, num_sms);
        default: return launch_unit_t<int64_t>(a, s, num_sms);
        }
    }
    return a.wide ? launch_o<Rec32>(a, s, num_sms) : launch_o<Rec16>(a, s, num_sms);
#endif
}

int k2_unit_words() { return kUnitWords; }
int k2_unit_max() { return kUnitMax; }
int k2_split_window() { return (int)(kBlockSmem / 8) / kGroup * kGroup; }
bool k2_block_regime(const K2Args &a) {
    const int words = a.pack16 ? 1 : 2;
    const int rcap = (a.R_max + kGroup - 1) / kGroup * kGroup;
    const size_t per_warp = (size_t)rcap * 4 * words;
    const int warps = (int)std::min<size_t>(8, (200 * 1024) / per_warp);
    return !(warps >= 2 && a.max_count <= 32768);
}

}  // namespace eucalc
