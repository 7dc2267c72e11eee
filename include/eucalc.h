/*
 * eucalc.h — C ABI of the B200-native exact Euler-characteristic, Radon and
 * hybrid transforms of weighted cubical complexes (arxiv 2405.02256).
 *
 * Citation keys: P:n = PAPER.md line n (the paper); S:n = SPEC.md line n.
 *
 * Conventions shared by every call
 * --------------------------------
 *  - Images are C-order (row-major, last axis fastest), axis i of the image
 *    <-> coordinate xi_i of a direction.
 *  - Directions are int32 [D][ndim], every coordinate nonzero (genericity,
 *    P:105). They may live on the host or the device.
 *  - Heights are integer LATTICE heights H = sum_i xi_i * (L/(M_i-1)) * p_i,
 *    p the vertex index, M_i the number of vertices on axis i, L the lcm of
 *    the (M_i - 1) > 0. The paper's normalised height (vertices evenly spaced
 *    in [-0.5,0.5]^n) is t = (2H - L*csum) / (2L) with csum the sum of
 *    xi_i over axes with M_i > 1: a strictly increasing map, so every order, tie
 *    and value is the paper's (E10). eucalc_height_map() returns L and csum.
 *  - Jumps use the TRUE right-minus-left sign J = chi(lower star) - chi(upper
 *    star) = -Delta^ord of P:87 (E1).
 *  - Pointers: every buffer argument may be host memory (pageable or pinned)
 *    or device memory; the library detects which with cudaPointerGetAttributes
 *    and copies as needed. All work is enqueued on `stream` (a cudaStream_t,
 *    NULL = legacy default stream). Calls that return host-visible results
 *    synchronise that stream, as documented per call.
 *  - Errors: no C++ exception crosses the ABI. On failure nothing is written
 *    to the outputs unless stated; eucalc_last_error() describes the failure
 *    (thread-local).
 */
#ifndef EUCALC_H
#define EUCALC_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum eucalc_status {
    EUCALC_OK = 0,
    EUCALC_E_ARG = 1,        /* bad dtype / ndim / shape / kernel / precision / NULL */
    EUCALC_E_NOMEM = 2,      /* device or host allocation failed */
    EUCALC_E_CUDA = 3,       /* a CUDA runtime error (see eucalc_last_error) */
    EUCALC_E_NONGENERIC = 4, /* a direction has a zero coordinate; see eucalc_last_bad_index */
    EUCALC_E_CAPACITY = 5,   /* an output buffer is too small; the required size is reported */
    EUCALC_E_RANGE = 6,      /* a height/value bound does not fit the requested element width */
    EUCALC_E_STATE = 7       /* invalid handle */
} eucalc_status;

enum { EUCALC_U8 = 0, EUCALC_I16 = 1, EUCALC_I32 = 2 };        /* image dtypes */
enum { EUCALC_VERTEX = 0, EUCALC_TOP = 1 };                    /* constructions */
enum { EUCALC_K_GAUSS = 0, EUCALC_K_COS = 1, EUCALC_K_SIN = 2, EUCALC_K_EXP = 3 };
enum { EUCALC_F32 = 0, EUCALC_F64 = 1 };

typedef struct eucalc_complex eucalc_complex;
typedef struct eucalc_critical eucalc_critical;

/* A batch of exact step-function representations in CSR form.
 * Segment s = image * D + direction holds entries [offsets[s], offsets[s+1]):
 * heights ascending (int lattice heights, see above) and the values there.
 * The value left of the first height is 0 (implicit leading E[0] = 0).
 * offsets: int64 [batch*D + 1]; height/value: int16, int32 or int64 [capacity]
 * (elem_bytes 2, 4 or 8). All three caller-owned. */
typedef struct eucalc_steps {
    int64_t *offsets;
    void *height;
    void *value;
    int64_t capacity;   /* entries available in height[] and value[] */
    int32_t elem_bytes; /* 2, 4 or 8 */
    int32_t reserved;   /* must be 0 */
} eucalc_steps;

/* ---- build (P:116 top-cell construction, P:140 dual/vertex construction) ----
 * img: `batch` same-shape images, C-order, dtype EUCALC_U8/I16/I32, host or
 * device. ndim 2 or 3; shape[ndim] >= 1. The image is copied: a HOST image may
 * be freed or reused as soon as the call returns (from pinned memory the call
 * waits for its copy); a DEVICE image must stay unchanged until the copy, which
 * is enqueued on `stream`, has run. The handle is library-owned
 * (eucalc_destroy_complex). EUCALC_U8: asynchronous for device images (|w| <= 255
 * by type); I16/I32: synchronises `stream` once (reads back max |weight|, used to
 * pick the record width).
 * Errors: E_ARG (dtype/ndim/shape/batch, packed vertex coords need > 32 bits),
 * E_NOMEM, E_CUDA. */
eucalc_status eucalc_build_complex(const void *img, int dtype, int ndim, const int64_t *shape,
                                   int64_t batch, int construction, void *stream,
                                   eucalc_complex **out);
/* Destroy calls free device memory stream-ordered on the stream the handle was
 * created on, after the work that any other stream enqueued with the handle so
 * far (the library records those streams). Every such stream must still exist
 * when the handle is destroyed. */
eucalc_status eucalc_destroy_complex(eucalc_complex *cx);

/* ---- critical points ----
 * For every image, vertex x and sign vector eps: Delta^-(eps,x) =
 * chi(phi|lwst), J(eps,x) = Delta^-(eps,x) - Delta^-(-eps,x) (E1; the
 * upper star w.r.t. eps is the lower star w.r.t. -eps). Vertices with
 * Delta^-(eps,x) != 0 or Delta^-(-eps,x) != 0 are kept, per antipodal pair
 * {eps,-eps}, in a deterministic order. The handle keeps a reference to `cx`
 * (destroy the critical handle first). Asynchronous. Errors: E_STATE, E_NOMEM, E_CUDA. */
eucalc_status eucalc_critical_points(const eucalc_complex *cx, void *stream, eucalc_critical **out);
eucalc_status eucalc_destroy_critical(eucalc_critical *cr);

/* h_counts: host int64 [batch][2^ndim][2] = (N^-, N^ord) per image and orthant
 * index e (bit i set iff eps_i = +1). Synchronises `stream`. */
eucalc_status eucalc_critical_counts(const eucalc_critical *cr, int64_t *h_counts, void *stream);

/* h_len: host int64 [batch][2^(ndim-1)] = length of each antipodal-pair list
 * (pair q = orthant index with bit ndim-1 clear). Synchronises `stream`. */
eucalc_status eucalc_critical_list_lengths(const eucalc_critical *cr, int64_t *h_len, void *stream);

/* Export the critical list of (image, orthant e): every kept vertex of e's
 * antipodal pair, with its row-major vertex id, Delta^-(e,x) and J(e,x).
 * Records with both zero cannot occur; records with Delta^- = 0 (not classical
 * for e) or J = 0 (not ordinary) can. Order: ascending vertex id.
 * vertex/dminus/jump: caller-owned, host or device, `cap` entries; *n_out gets
 * the list length. Synchronises `stream`. E_CAPACITY if cap < length (nothing written). */
eucalc_status eucalc_critical_export(const eucalc_critical *cr, int64_t image, int orthant,
                                     int64_t *vertex, int32_t *dminus, int32_t *jump,
                                     int64_t cap, int64_t *n_out, void *stream);

/* Upper bounds of the total number of entries of the ECT (= classical Radon)
 * and ordinary Radon outputs for these directions: sum over (image, direction)
 * of min(list length, height range R). Synchronises `stream` on first use. */
eucalc_status eucalc_output_bound(const eucalc_critical *cr, const int32_t *dirs, int64_t D,
                                  int64_t *bound_ect, int64_t *bound_ordinary, void *stream);
/* A looser bound that needs no K1 result and never synchronises: sum over
 * (image, direction) of min(vertices, height range R) (a list holds at most one
 * record per vertex). Any capacity >= eucalc_output_bound() is accepted by
 * eucalc_transforms, so a caller can allocate with this bound while K1 still
 * runs. dirs: host pointer (device pointers synchronise to read them).
 * Errors: E_NONGENERIC, E_ARG. */
eucalc_status eucalc_output_bound_upper(const eucalc_complex *cx, const int32_t *dirs, int64_t D,
                                        int64_t *bound, void *stream);

/* ---- exact transforms (Lemma 2) ----
 * For every (image, direction):
 *   ect       : (T, E)     ECT(xi,t) = sum_{classical x} Delta^- 1[t >= h(x)]
 *   ordinary  : (T_o, E')  heights where Radon(t+) != Radon(t-), value Radon(t+) (E1)
 *   classical : (T_c, E_c) heights where Radon(t) != Radon(t-), value Radon(t)   (E7)
 * Equal heights are merged and zero-net entries dropped (canonical form, E8).
 * Any of ect/ordinary/classical may be NULL (not computed). A classical
 * `height` pointer equal to the ect `height` pointer is written once (T_c = T).
 * Capacity: each non-NULL output must hold eucalc_output_bound() entries
 * (ect/classical: bound_ect, ordinary: bound_ordinary), else E_CAPACITY with
 * *required_out (if non-NULL) = that bound and nothing written. Element widths
 * 2 and 4 are accepted when every height and value provably fits int16 / int32
 * (host-checked bounds from K1's statistics), else E_RANGE; E_RANGE also when
 * batch * D >= 2^31 segments or the total output exceeds 2^31 entries.
 * The exact total of segment s is offsets[s+1] - offsets[s].
 * Device outputs: asynchronous except the first bound query. Host outputs:
 * computed into library scratch and copied back, then `stream` is synchronised.
 * Errors: E_NONGENERIC (eucalc_last_bad_index() = first bad direction),
 * E_CAPACITY, E_RANGE, E_ARG, E_NOMEM, E_CUDA. */
eucalc_status eucalc_transforms(const eucalc_critical *cr, const int32_t *dirs, int64_t D,
                                eucalc_steps *ect, eucalc_steps *ordinary, eucalc_steps *classical,
                                int64_t *required_out, void *stream);
/* eucalc_transforms plus the hybrid transform of every (image, direction) from
 * the same merged height histogram (NEXT row f2): HT(xi) = -sum_h H_J(h) kbar(t(h)),
 * H_J(h) the sum of J over the critical points at lattice height h — Lemma 2's
 * sum with equal heights grouped, so one kbar (tabulated per lattice
 * u, E21) per distinct height instead of one per ordinary point. kernel, param,
 * precision and ht_out ([batch][D], host or device) as for eucalc_hybrid; the
 * ordinary stream must be requested. Deterministic (fixed-order sums). When
 * the kbar table would exceed 2^24 entries (unequal extents make L, hence the
 * u range, large) the HT is computed by eucalc_hybrid after the transforms
 * instead (same tolerance). Errors as for eucalc_transforms and eucalc_hybrid. */
eucalc_status eucalc_transforms_ht(const eucalc_critical *cr, const int32_t *dirs, int64_t D,
                                   eucalc_steps *ect, eucalc_steps *ordinary, eucalc_steps *classical,
                                   int kernel, double param, int precision, void *ht_out,
                                   int64_t *required_out, void *stream);
/* ---- real-valued directions (NEXT row f3; the paper's setting) ----
 * dirs: double [D][ndim] (host or device), finite, every coordinate nonzero
 * (E_NONGENERIC otherwise). A vertex p is embedded at
 * x_i = p_i/(M_i-1) - 0.5 (0 when M_i = 1) and its height is the double
 * ((xi_0 x_0 + xi_1 x_1) + xi_2 x_2) + 0.0 computed left to right in IEEE
 * double, round to nearest, no fused multiply-add; equal heights are equal
 * computed dots (E22). Breakpoints are sorted (the paper's
 * sort + merge) per (image, direction). Outputs as for
 * eucalc_transforms, with height[] double and value[] int64: elem_bytes must
 * be 8. Capacity: sum over (image, direction) of the list length (reported in
 * *required_out). Any list length: lists of <= 4096 records are sorted by one
 * warp in shared memory; longer lists take a bucketed path (value buckets of
 * ~128 records, each sorted by a warp or, when oversize, by a CTA, then merged
 * with running sums), processed in chunks whose device scratch (32 B per record)
 * stays within min(free memory / 4, 8 GiB); E_NOMEM if one segment alone does
 * not fit. Host outputs synchronise `stream`. */
eucalc_status eucalc_transforms_real(const eucalc_critical *cr, const double *dirs, int64_t D,
                                     eucalc_steps *ect, eucalc_steps *ordinary, eucalc_steps *classical,
                                     int64_t *required_out, void *stream);
eucalc_status eucalc_ect(const eucalc_critical *cr, const int32_t *dirs, int64_t D,
                         eucalc_steps *ect, int64_t *required_out, void *stream);
eucalc_status eucalc_radon(const eucalc_critical *cr, const int32_t *dirs, int64_t D,
                           eucalc_steps *ordinary, eucalc_steps *classical,
                           int64_t *required_out, void *stream);

/* ---- hybrid transform (Lemma 2) ----
 * HT(xi) = int kappa(t) Radon(xi,t) dt = -sum_{ordinary x} J(eps,x) kbar(t(x)),
 * t the paper's normalised height. Kernels (kappa -> kbar):
 *   GAUSS: exp(-t^2/(2 s^2)) -> s sqrt(pi/2) erf(t/(s sqrt 2)),  param = s > 0
 *   COS  : cos(2 pi t / P)   -> P/(2 pi) sin(2 pi t / P),       param = P > 0
 *   SIN  : sin t             -> -cos t,               param ignored
 *   EXP  : exp t             -> exp t   (Appendix A),   param ignored
 * out: [batch][D] float (F32) or double (F64), host or device, caller-owned.
 * Deterministic: identical bits run to run (fixed-order combine).
 * Errors: E_NONGENERIC, E_ARG, E_NOMEM, E_CUDA. */
eucalc_status eucalc_hybrid(const eucalc_critical *cr, const int32_t *dirs, int64_t D, int kernel,
                            double param, int precision, void *out, void *stream);

/* eucalc_hybrid with an explicit algorithm (eucalc_hybrid = EUCALC_HT_AUTO):
 *   EUCALC_HT_DIRECT: kbar evaluated per (ordinary point, direction) term;
 *   EUCALC_HT_TABLE : kbar depends on a term only through the integer
 *     u = 2H - L*csum (E10), so it is evaluated once per u in fp64 and looked up
 *     (same values as DIRECT up to the final rounding of kbar to the output
 *     precision). Needs packed byte-aligned coordinates (extents <= 65536 in
 *     2-D, <= 256 in 3-D), axis-scaled |xs_i| <= 127 and a u-range whose half
 *     table fits shared memory, else E_ARG;
 *   EUCALC_HT_AUTO  : TABLE when it applies, else DIRECT. */
enum { EUCALC_HT_AUTO = 0, EUCALC_HT_DIRECT = 1, EUCALC_HT_TABLE = 2 };
eucalc_status eucalc_hybrid_ex(const eucalc_critical *cr, const int32_t *dirs, int64_t D, int kernel,
                               double param, int precision, int algorithm, void *out, void *stream);

/* ---- evaluation and vectorisation (P:135-137 evaluation, P:339-341 vectorisation) ----
 * Values of exact representations at real heights t, given in the paper's
 * normalised units (vertices evenly spaced in [-0.5,0.5]^n):
 *   kind EUCALC_EVAL_ECT  : ECT(xi,t) = E at the last breakpoint with height <= t,
 *                           0 before the first;
 *   kind EUCALC_EVAL_RADON: Radon(xi,t) = E_c if t equals a classical height
 *                           (P:137), else E' at the last ordinary breakpoint
 *                           strictly below t (E7), 0 before the first.
 * Every comparison t(H) <= t / < t / == t is decided exactly (t is mapped to
 * lattice units with an error-free product, E20), so the results are
 * those of the definitions at the double t. t = +-inf is allowed; a NaN query
 * yields 0.
 * cx, dirs, D: the complex and the directions the representations were computed
 *   for (segment s = image*D + direction, as produced by eucalc_transforms).
 * rep: the ECT stream (ECT) or the ordinary Radon stream (T_o, E') (Radon);
 * classical: the classical Radon stream (T_c, E_c) (Radon; NULL for ECT).
 *   The classical height pointer may alias the ECT heights (T_c = T).
 *   Host or device; elem_bytes 2, 4 or 8 (shared by rep and classical).
 * eucalc_evaluate : queries t[nq] (host or device doubles), the same for every segment.
 * eucalc_vectorize: the N evenly spaced points t_i = a + (i*(b-a))/(N-1),
 *   i = 0..N-1 (t_0 = a when N = 1), computed in IEEE double round-to-nearest
 *   in that order.
 * out: [batch*D][nq or N] int32 or int64 (out_elem_bytes 4 or 8; 4 requires
 *   the representation's elem_bytes <= 4), host or device, caller-owned.
 * Asynchronous for device buffers; host buffers synchronise `stream`.
 * Errors: E_ARG (NULL/shape/elem_bytes/kind), E_NONGENERIC, E_NOMEM, E_CUDA. */
enum { EUCALC_EVAL_ECT = 0, EUCALC_EVAL_RADON = 1 };
eucalc_status eucalc_evaluate(const eucalc_complex *cx, const int32_t *dirs, int64_t D, int kind,
                              const eucalc_steps *rep, const eucalc_steps *classical,
                              const double *t, int64_t nq, void *out, int out_elem_bytes, void *stream);
eucalc_status eucalc_vectorize(const eucalc_complex *cx, const int32_t *dirs, int64_t D, int kind,
                               const eucalc_steps *rep, const eucalc_steps *classical,
                               double a, double b, int64_t N, void *out, int out_elem_bytes, void *stream);

/* ---- helpers ---- */
/* L and csum of the height map t = (2H - L*csum)/(2L) for direction dir (host, [ndim]). */
eucalc_status eucalc_height_map(const eucalc_complex *cx, const int32_t *dir, int64_t *L, int64_t *csum);
/* Stage timing with CUDA events recorded on the launching stream around each
 * kernel group: stages "build", "k1_critical", "k2_transforms", "k3_hybrid".
 * eucalc_profile_enable(1) clears and starts recording on the calling thread,
 * (0) stops. eucalc_profile_read synchronises the recorded events and returns
 * the summed milliseconds and number of recorded launches of `stage`. */
void eucalc_profile_enable(int on);
int eucalc_profile_read(const char *stage, double *ms, int64_t *launches);
/* Wall span (first start to last end, milliseconds) of the recorded launches of
 * `stage`, which may run concurrently on several streams. Synchronises them. */
int eucalc_profile_span(const char *stage, double *ms);
/* Kernel launches issued by this library on the calling thread since the last reset. */
int64_t eucalc_launch_count(int reset);
/* Diagnostic (tests): K2 block-regime segments whose checked packed histogram
 * bins flagged a possible field overflow and were recomputed with split bins,
 * since the last reset. Counted only while the EUCALC_K2_CHK_BITS test hook is
 * set (the count is read back after each such call, which synchronises it). */
int64_t eucalc_k2_restarts(int reset);
const char *eucalc_status_string(eucalc_status s);
const char *eucalc_last_error(void);
int64_t eucalc_last_bad_index(void);

#ifdef __cplusplus
}
#endif
#endif /* EUCALC_H */
