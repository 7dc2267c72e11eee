// Internal declarations shared by the eucalc CUDA translation units.
// Product code only: nothing here is shared with oracle/ (test infrastructure).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/eucalc.h"

// Device-side bounds checks (the stand-in for compute-sanitizer memcheck, which
// the GPU pool does not allow): built into libeucalc_checked.so only
// (_build.build(checked=True), -DEUCALC_DEVICE_CHECKS); a failed check prints
// the file and line and traps, so the launch (and the test) fails with E_CUDA.
#ifdef EUCALC_DEVICE_CHECKS
#include <cstdio>
#define EU_DCHECK(cond)                                                                        \
    do {                                                                                       \
        if (!(cond)) {                                                                         \
            printf("EU_DCHECK failed: %s:%d: %s (block %d thread %d)\n", __FILE__, __LINE__, #cond, \
                   (int)blockIdx.x, (int)threadIdx.x);                                         \
            __trap();                                                                          \
        }                                                                                      \
    } while (0)
#else
#define EU_DCHECK(cond) ((void)0)
#endif

namespace eucalc {

constexpr int kMaxN = 3;

// One record of a critical list: packed vertex coordinates + Delta^- for the
// pair's representative orthant (a) and for its antipode (b). SURVEY 8(a) A2.
struct __align__(8) Rec16 {
    uint32_t c;
    int16_t a, b;
};
struct Rec32 {
    uint32_t c;
    int32_t a, b;
};

// ---- host-side handles -----------------------------------------------------
// Streams other than the owner stream that enqueued work reading a handle's
// device memory: the destroy call orders its stream-ordered frees after them.
struct StreamSet {
    std::mutex mu;
    std::vector<cudaStream_t> v;
    void note(cudaStream_t s, cudaStream_t owner) {
        if (s == owner) return;
        std::lock_guard<std::mutex> lk(mu);
        if (std::find(v.begin(), v.end(), s) == v.end()) v.push_back(s);
    }
    // makes `owner` wait for the work enqueued so far on every noted stream
    void join(cudaStream_t owner) {
        std::lock_guard<std::mutex> lk(mu);
        for (cudaStream_t s : v) {
            cudaEvent_t e;
            if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) continue;
            if (cudaEventRecord(e, s) == cudaSuccess) cudaStreamWaitEvent(owner, e, 0);
            cudaEventDestroy(e);
        }
        cudaGetLastError();
        v.clear();
    }
};

struct Complex {
    int ndim = 0, dtype = 0, construction = 0;
    int64_t batch = 0;
    int64_t m[kMaxN] = {1, 1, 1};  // image extents (pixels)
    int64_t M[kMaxN] = {1, 1, 1};  // vertex extents
    int64_t npix = 0, nvert = 0;   // per image
    void *d_img = nullptr;         // device copy, batch * npix elements
    int64_t max_abs_w = 0;
    int sh[kMaxN] = {0, 0, 0};     // packed coordinate shifts
    uint32_t msk[kMaxN] = {0, 0, 0};
    int aligned = 0;               // 2: 16-bit coordinate halves (dp2a), 3: bytes (dp4a), 0: generic
    int64_t L = 1;                 // lcm of (M_i - 1) > 0
    int64_t scale[kMaxN] = {0, 0, 0};
    cudaStream_t owner_stream = nullptr;
    StreamSet users;
};

struct Critical {
    const Complex *cx = nullptr;
    int Q = 0;          // antipodal pairs = 2^(n-1)
    bool wide = false;  // Rec32 instead of Rec16
    int64_t vcap = 0;   // records capacity per (image, pair) list = nvert
    void *d_rec = nullptr;       // [batch][Q][vcap]
    int32_t *d_count = nullptr;  // [batch][Q]
    int32_t *d_tile_off = nullptr;  // [batch][Q][ntiles+1] (K1 tile -> list offset)
    int TX = 1, TY = 1, TZ = 1, tiles_x = 1, tiles_y = 1, tiles_z = 1, ntiles = 1;
    int64_t *d_stats = nullptr;  // [batch][2^n][2] (N^-, N^ord), [batch][Q] sum(|a|+|b|), [batch][Q] max(|a|+|b|)
    // host cache (filled by sync_counts)
    bool have_host = false;
    int64_t *h_count = nullptr;  // [batch][Q]
    int64_t *h_stats = nullptr;
    int64_t max_count = 0;
    int64_t max_abs_sum = 0;
    int64_t max_rec = 0;
    std::mutex mu;            // guards the host caches below (concurrent read-only use)
    uint64_t bound_plan = 0;  // eucalc_output_bound cache: direction plan id -> bound
    int64_t bound_val = 0;
    cudaStream_t owner_stream = nullptr;
    StreamSet users;
    cudaEvent_t k1_done = nullptr;  // after the async read-back of counts/stats
    bool have_orthant_counts = false;  // N^-, N^ord computed (eucalc_critical_counts)
    void *pinned = nullptr;         // pinned host copy: int32 counts, then int64 stats
    size_t pinned_bytes = 0, pinned_stats_off = 0;
    size_t pinned_flag_off = 0;     // signal word (k1_signal) polled by sync_counts, 0 = none
};

// Pinned host memory pool (power-of-two size classes, reused; never unpinned).
void *pinned_get(size_t bytes, size_t *cap);
void pinned_put(void *p, size_t cap);

// ---- launchers (implemented in the .cu files) -------------------------------
struct K1Args {
    const void *img;
    int dtype, construction, ndim;
    int64_t batch, npix, vcap;
    int m[kMaxN], M[kMaxN];
    int TX, TY, TZ, tiles_x, tiles_y, tiles_z;
    int W;              // warps (pencils) per tile: 8 in 3-D (one per row), 1 in 2-D
    int walk;           // 3-D: planes walked per CTA (k1_walk)
    bool stats_in_copy; // the |Delta^-| statistics are taken by k1_copy (two-vertex 3-D pencils)
    int sh[kMaxN];
    void *rec;
    bool wide;
    int32_t *count;
    int32_t *tile_off;  // [batch][Q][ntiles+1] list offset of each tile (+ total)
    int32_t *cnt;       // [batch][Q][ntiles][W] kept counts -> (scan) offsets (zeroed)
    void *scratch;      // [batch][Q][scap] records in fixed-capacity (tile, warp) regions
    int64_t scap;       // scratch records per list = ntiles * W * cap_r
    int cap_r;          // records per region = vertices of one (tile, warp)
    int Q;
    bool direct;        // one region per image: records go straight to the lists
    unsigned long long *flags;  // [k1_scan_chunks] scan look-back flags (zeroed)
    unsigned int *ticket;       // scan chunk ticket (zeroed)
    int64_t *stats;     // [batch][2^n][2] N^-, N^ord (on demand: launch_k1_stats)
    int64_t *abs_sum;
    int64_t *max_rec;
};
// K1 tile geometry for an image of ndim dims (vertex extents M).
void k1_geometry(int ndim, const int64_t *M, int dtype, int construction, int *TX, int *TY, int *TZ, int *W);
// 3-D: planes walked per K1 CTA for a batch of images
int k1_walk(int ndim, const int64_t *M, int64_t batch, int TX, int TY);
// Look-back flags k1_scan needs for `lists` lists of ntiles * W counts.
int64_t k1_scan_chunks(int64_t lists, int64_t ntiles, int W);
cudaError_t launch_k1(const K1Args &a, cudaStream_t s);
cudaError_t launch_k1_stats(const K1Args &a, cudaStream_t s);

// Per-direction info for K2/K3 (host-computed, copied to device).
struct DirInfo {
    int xs[kMaxN];  // axis-scaled direction xi_i * L/(M_i-1)
    int hlo;        // lowest lattice height
    int R;          // number of lattice heights
    int q;          // antipodal pair of the orthant
    int swap;       // 1 if the orthant is the pair's non-representative
    int xs8;        // xs as packed int8 (byte j <-> axis n-1-j) when every |xs_i| <= 127
    int line;       // max vertices on one lattice height level (bounds every bin's record count)
    long long lcsum;  // L * csum (u = 2H - L*csum, the kbar table argument of the fused HT)
};

struct StepsOut {
    int64_t *off;
    void *h;
    void *v;
};

struct K2Args {
    const void *rec;
    bool wide;
    int64_t vcap;
    const int32_t *count;
    int Q, ndim;
    int sh[kMaxN];
    uint32_t msk[kMaxN];
    const DirInfo *dirs;
    int64_t D, batch;
    int R_max;
    int64_t max_count;
    int elem_bytes;
    int dp;       // 2/3: heights by dp2a/dp4a on byte-aligned coordinates; 0: shifts and masks
    bool pack16;  // 16+16-bit packed histogram bins are exact (host-checked)
    bool do_ect, do_ord, do_cls, cls_alias;
    StepsOut ect, ord, cls;
    const int32_t *tile_off;    // [batch][Q][ntiles+1] K1 tile -> list offset
    int ntiles, tiles_x, tiles_y, TX, TY, TZ;
    int M[kMaxN];               // vertex extents
    unsigned long long *flags;  // [batch*D] look-back flags (zeroed)
    unsigned int *ticket;       // [4] ticket counters (zeroed)
    int *cnt_c, *cnt_o;         // [batch*D] per-segment counts (warp regime)
    uint2 *slab;                // [batch*D][33] merged runs of lists <= sparse_max records, or NULL
    int sparse_max;             // lists of <= sparse_max (<= 32) records: register sort instead of histogram
    bool sum16;                 // every list's sum |a|+|b| < 2^15: (wj, wc) prefix sums fit packed 16+16 bits
    int64_t max_rec, max_abs_sum;  // K1 statistics: max |a|+|b| of a record, max list sum of |a|+|b|
    bool no_chk;                // block regime: never use checked packed bins (EUCALC_K2_NO_CHK, tests)
    unsigned chk_bias, chk_mask;  // checked packed bins: fields in [-2^k, 2^k), k = 14 (EUCALC_K2_CHK_BITS, tests)
    void *stage;                // block regime: per-CTA output staging (k2_stage_bytes), or NULL
    int64_t stage_cap;          // entries per staged array per CTA (unit path: per image batch, all segments)
    // unit path (k2_unit): several directions per pass over a list, or units == NULL
    const int4 *units;          // [nunits] {first index into unit_dirs, G, pair q, swap}, one image's units
    int64_t nunits;
    const int32_t *unit_dirs;   // direction ids of the units
    const int64_t *stage_base;  // [D] staging slot of direction d within an image (prefix of R)
    int64_t stage_img;          // staging entries per image (sum of R)
    const int32_t *img_order;   // [batch] images by decreasing list size (all units of the heaviest image first), or NULL
    const int32_t *seg_order;   // [D] slot mode: directions by decreasing R (longest segments first), or NULL
    // fused HT (NEXT f2): kbar table (fp64) over u in [ht_U0, ...), or NULL
    const double *ht_tab;
    int64_t ht_U0, L;
    int64_t ht_U;               // table length
    const int32_t *csum;        // [D]
    double ht_scale;            // HT = ht_scale * sum_h H_J(h) f(u(h))
    int ht_prec;
    void *ht_out;               // [batch][D]
    int64_t out_cap;            // entries every requested output array holds (device checks)
};
cudaError_t launch_k2(const K2Args &a, cudaStream_t s, int num_sms);
// unit path geometry: packed histogram words per CTA, directions per unit, split window
int k2_unit_words();
int k2_unit_max();
int k2_split_window();
// the block regime (one CTA per segment / unit) is taken for these arguments
bool k2_block_regime(const K2Args &a);
// Block regime only: bytes of per-CTA output staging that let each segment fill
// its histogram once (0 = warp regime, or staging too large: two fills).
size_t k2_stage_bytes(const K2Args &a, int num_sms, int64_t *cap);

struct K3Args {
    const void *rec;
    bool wide;
    int64_t vcap;
    const int32_t *count;
    int Q, ndim;
    int sh[kMaxN];
    uint32_t msk[kMaxN];
    const DirInfo *dirs;       // per direction (original order)
    const int32_t *order;      // sorted direction index list (grouped by orthant)
    const int32_t *tile_start; // [ntiles] start into order; tile = same-orthant, same-parity run of <= 512
    const int32_t *tile_len;
    int ntiles;
    int64_t D, batch;
    int kernel, precision;
    double param;
    int64_t L;
    const int32_t *csum;       // [D] sum of xi_i over axes with M_i > 1
    int dp;                    // as K2Args::dp
    int threads;               // block size = longest tile rounded up to a warp
    int nchunks;
    int chunk;                 // records per CTA
    double *partial;           // [batch][nchunks][D]
    void *out;                 // [batch][D]
    // tabulated kbar (use_table): u = 2H - L*csum in [U0, U0 + U)
    int use_table;
    int64_t U0, U;
    double *tab64;
    float *tab32;
};
int k3_chunk(bool table);
int k3_mode(int kernel, int precision, bool wide);
size_t k3_table_smem(int mode, long long U);
cudaError_t launch_k3(const K3Args &a, cudaStream_t s);
// kbar table for u in [U0, U0 + U) in fp64, parity-split (even u - U0 first, then
// odd; K2's fused HT), with an optional fp32 copy in natural order; and the HT
// scale of each kernel
cudaError_t launch_k3_table_only(int kernel, double param, int64_t L, int64_t U0, int64_t U, double *t64, float *t32,
                                 cudaStream_t s);
double k3_scale(int kernel, double param);

// K4: evaluation / vectorisation (NEXT f1)
struct K4Args {
    int kind;                   // EUCALC_EVAL_ECT / EUCALC_EVAL_RADON
    const int64_t *rep_off;     // [batch*D+1] ECT or ordinary Radon stream
    const void *rep_h, *rep_v;
    const int64_t *cls_off;     // classical Radon stream (Radon only)
    const void *cls_h, *cls_v;
    int in_eb, out_eb;
    int64_t L;
    const int32_t *csum;        // [D]
    int64_t D, batch;
    const double *t;            // [nq] queries, or NULL: t_i = ta + (i*(tb-ta))/(nq-1)
    double ta, tb;
    int64_t nq;
    void *out;                  // [batch*D][nq]
};
cudaError_t launch_k4(const K4Args &a, cudaStream_t s, int num_sms);

// Launch preparation with a per-process cache: the dynamic shared memory
// attribute is raised to the largest `smem` seen for `fn` and the occupancy
// (blocks per SM at `threads`, `smem`) is memoised, so the host cost of a
// repeated launch is a map lookup instead of two driver calls.
cudaError_t prepare_kernel(const void *fn, int threads, size_t smem, int *occ);

// CSR offsets from per-segment counts (K2's decoupled-look-back scan): writes
// a.ect/cls/ord.off[0..S] for the requested streams; a.ticket[2] and a.flags
// (S entries) must be zeroed.
cudaError_t launch_csr_scan(const K2Args &a, const int *cnt_c, const int *cnt_o, long long S, cudaStream_t s);

// K5: real-valued directions (NEXT f3)
struct K5Args {
    const void *rec;
    bool wide;
    int64_t vcap;
    const int32_t *count;
    int Q, ndim;
    int sh[kMaxN];
    uint32_t msk[kMaxN];
    int M[kMaxN];
    const double *xi;     // [D][ndim]
    const int32_t *q;     // [D] antipodal pair of the direction's orthant
    const int32_t *swap;  // [D] 1 if the orthant is the pair's non-representative
    int64_t D, batch;
    int npow2;            // sort length: power of two >= every small list length
    int small_max;        // lists longer than this take the bucketed path (K5Big)
    int *cnt_c, *cnt_o;   // [batch*D]
    bool do_ect, do_ord, do_cls, cls_alias;
    StepsOut ect, ord, cls;  // heights double, values int64
    K2Args scan;          // offsets / ticket / flags for launch_csr_scan
};
// Bucketed path for lists longer than small_max (one chunk of big segments):
// value buckets -> pieces (contiguous in scratch, equal heights never split),
// each piece sorted (warp bitonic, or a CTA sort for oversize pieces) and
// run-length merged with the running sums of the pieces before it.
struct K5Big {
    const int64_t *seg;    // [nseg] segment ids s = b*D + d, ascending
    const int64_t *pbase;  // [nseg] first piece (chunk-local)
    const int32_t *nb;     // [nseg] buckets (= pieces) of the segment
    const int64_t *sbase;  // [nseg] first scratch record
    int64_t nseg, npieces;
    uint4 *scr, *tmp;      // records {key lo, key hi, Delta^-, J}, and merge-sort ping-pong
    int64_t *p_start;      // [npieces] first scratch record
    int32_t *p_len, *p_seg;
    int32_t *p_nc, *p_no, *p_sc, *p_sj;      // run counts and sums per piece
    int32_t *p_offc, *p_offo, *p_ic, *p_ij;  // exclusive within the segment
    unsigned *over;        // [0] oversize pieces, [1] ticket, then the list from over+2
    int64_t over_cap;
};
constexpr int kK5PieceMax = 512;    // pieces up to this many records: warp sort in smem
constexpr int kK5Bucket = 128;      // target records per bucket
constexpr int kK5MaxBuckets = 32768;
// phase 0: counts, 1: emit (small lists only; big segments are skipped)
cudaError_t launch_k5(const K5Args &a, int phase, cudaStream_t s, int num_sms);
cudaError_t launch_k5_scan(const K5Args &a, cudaStream_t s);
// bucket + sort + per-piece counts + segment scan (writes cnt_c/cnt_o of its segments)
cudaError_t launch_k5b_prepare(const K5Args &a, const K5Big &g, int nb_max, cudaStream_t s, int num_sms);
cudaError_t launch_k5b_emit(const K5Args &a, const K5Big &g, cudaStream_t s, int num_sms);
size_t k5_smem(int npow2);

// thread-local launch counter (eucalc_launch_count)
void count_launch(int n = 1);

}  // namespace eucalc
