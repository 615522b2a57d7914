/*
 * hexval.h -- C ABI of the B200 hot path for the robust validity check of
 * linear hexahedra (Johnen, Weill, Remacle, "Robust and efficient validation
 * of the linear hexahedral element", IMR26 2017 = /root/reference/PAPER.md).
 *
 * Problem statement: "takes the coordinates of 8
 * points as input and outputs the validity of the hexahedron".  A hexahedron
 * is VALID iff its Jacobian determinant det J is strictly positive on the
 * whole reference cube [0,1]^3 (Eq. e:det3d 416-423).
 *
 * Per hex the library runs the algorithm of PAPER.md section 6
 * (lines 1105-1145):
 *   1. the 20 Jacobian samples (8 corners, 12 edge midpoints) as tetrahedron
 *      determinants (section 5);
 *   2. any sample <= 0 -> INVALID (samples within their rounding bound of 0
 *      are decided in exact arithmetic, reading G8);
 *   3. the 27 Bezier coefficients b = T~ c20 (Table 3);
 *   4. all of b_9..b_27 > 0 -> VALID;
 *   5. otherwise recursive_subdivision(b): de Casteljau octree subdivision,
 *      depth cap HEXVAL_MAX_DEPTH (children at that depth are classified but
 *      not split; an undecided one makes the hex UNDETERMINED).
 *
 * Everything runs on one CUDA device in hand-written sm_100a kernels; there
 * is no CPU fallback.  All entry points are plain C: host/device pointers,
 * sizes and a cudaStream_t (no framework types).
 */
#ifndef HEXVAL_H
#define HEXVAL_H

#include <stdint.h>
#include <cuda_runtime_api.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (return values; never thrown) ------------------------ */
#define HEXVAL_OK               0
#define HEXVAL_ERR_ARGUMENT    (-1)  /* n < 0, n > INT32_MAX, or NULL with n > 0 */
#define HEXVAL_ERR_ALIGNMENT   (-2)  /* a double/int pointer not 8/4-byte aligned */
#define HEXVAL_ERR_CUDA        (-3)  /* launch / configuration / copy error */
#define HEXVAL_ERR_ALLOC       (-4)  /* scratch allocation failed */

/* ---- per-hex flags byte ----------------------------------------------------
 * bits 0-1: verdict, bit 2: SUBDIVIDED (root undecided after Step 4, i.e.
 * recursive_subdivision was entered), bits 3-7: zero.                       */
#define HEXVAL_INVALID          0
#define HEXVAL_VALID            1
#define HEXVAL_UNDETERMINED     2    /* depth cap reached, no INVALID found  */
#define HEXVAL_NONFINITE        3    /* a coordinate is NaN/Inf or |x| > 2^300 */
#define HEXVAL_FLAG_SUBDIVIDED  4
#define HEXVAL_MAX_DEPTH        20

/* Device-side counters, accumulated with atomics when a pointer is passed to
 * the *_ex calls.  The caller allocates it in device memory and zeroes it. */
typedef struct hexval_stats {
    unsigned long long n_valid;          /* final verdict counts            */
    unsigned long long n_invalid;
    unsigned long long n_undetermined;
    unsigned long long n_nonfinite;
    unsigned long long n_subdivided;     /* hexes with SUBDIVIDED set       */
    unsigned long long n_exact;          /* hexes whose Step 2 needed exact signs */
    unsigned long long n_nodes;          /* recursive_subdivision calls     */
    unsigned long long max_depth;        /* deepest child depth classified  */
    unsigned long long n_lane_steps;     /* subdivision kernel: 32 x warp steps (lane slots
                                            offered); n_nodes / n_lane_steps = lane use */
} hexval_stats;

/* Per-phase kernel timing (CUDA events recorded on the call's stream). */
typedef struct hexval_profile hexval_profile;
#define HEXVAL_PHASE_PASS1   0   /* pass-1 kernel: 20 dets, 27 coeffs, classify, compact */
#define HEXVAL_PHASE_EXACT   1   /* exact signs: fused into the subdivision kernel, reads 0 */
#define HEXVAL_PHASE_SUBDIV  2   /* subdivision kernel                                   */
#define HEXVAL_NUM_PHASES    3

/* ---- device-resident calls (asynchronous) ----------------------------------
 * coords       SoA, 24 planes of n doubles: coords[(3*k + a)*n + i] is axis a
 *              (x,y,z) of node k = 0..7 of hex i, nodes in Fig. 3 order
 *              (bottom face 1-2-3-4 counter-clockwise, then
 *              top face 5-6-7-8).  Device memory, 8-byte aligned.
 * vertices     AoS xyz, vertices[3*v + a]; device memory, 8-byte aligned.
 * hex_idx      row-major int32 [n][8] vertex ids in Fig. 3 order; device
 *              memory, 4-byte aligned.  Precondition: 0 <= id < number of
 *              vertices (not checked; there is no nv argument).
 * flags_out    n bytes, device memory (see flags above).
 * coeffs_out_opt  NULL or 27*n doubles, device memory, coefficient-major:
 *              coeffs[s*n + i] = b_{s+1} of hex i in Fig. 3 order (b_1..8
 *              corners, 9..20 edges, 21..26 faces, 27 centre), the Bezier
 *              coefficients of det J (det J, i.e. 6 x volume, not volumes).
 *              Written for every hex (also INVALID ones); unspecified for
 *              NONFINITE hexes.
 * stream       CUDA stream; all work is enqueued on it, results are valid
 *              after the stream synchronises.  No host synchronisation
 *              happens inside the call.  Calls on different streams are
 *              independent: scratch (control block, work queues, the
 *              subdivision stacks) is borrowed from persistent library-owned
 *              arenas, one per stream with calls in flight, stream-ordered
 *              (see hexval_scratch_info); steady-state calls allocate nothing.
 * Device       the calling thread's current device (cudaSetDevice): every
 *              device buffer and the stream must belong to it.
 * Ownership    the caller owns every buffer; the library never frees them.
 * n == 0       returns HEXVAL_OK without enqueueing work.
 * Returns      HEXVAL_OK or a negative status (see above).  Data problems
 *              (NaN/Inf, out of range) are per-hex flags, never a status.   */
int hexval_check_soa(const double* coords, int64_t n, uint8_t* flags_out,
                     double* coeffs_out_opt, cudaStream_t stream);

int hexval_check_indexed(const double* vertices, const int32_t* hex_idx, int64_t n,
                         uint8_t* flags_out, double* coeffs_out_opt, cudaStream_t stream);

/* Same, plus optional device stats (accumulated) and optional profile. */
int hexval_check_soa_ex(const double* coords, int64_t n, uint8_t* flags_out,
                        double* coeffs_out_opt, hexval_stats* stats_dev_opt,
                        hexval_profile* profile_opt, cudaStream_t stream);

int hexval_check_indexed_ex(const double* vertices, const int32_t* hex_idx, int64_t n,
                            uint8_t* flags_out, double* coeffs_out_opt,
                            hexval_stats* stats_dev_opt, hexval_profile* profile_opt,
                            cudaStream_t stream);

/* Steps 4-5 alone on caller-supplied Bezier coefficient
 * vectors: coeffs is device memory, coefficient-major coeffs[s*n + i] (Fig. 3
 * order, as coeffs_out above).  Item i is VALID if all of b_9..27 > 0, else
 * recursive_subdivision runs on it (flags as above, SUBDIVIDED set).  As in the
 * paper, Step 4 presumes the corner coefficients b_1..8 were already checked
 * (they are only tested again as children's corners).  An item with a NaN/Inf
 * coefficient gets NONFINITE.  Used for quality queries on arbitrary
 * triquadratics and to pin the subdivision kernel in the tests.            */
int hexval_classify_bezier(const double* coeffs, int64_t n, uint8_t* flags_out,
                           hexval_stats* stats_dev_opt, cudaStream_t stream);

/* ---- NEXT-2: screening by-products of the 8 corner samples ---------------------
 * For every hex (layouts as above; outputs are device memory, either may be NULL):
 *   sj_min_out_opt[i]  min over the 8 corners of the scaled Jacobian
 *                      det J / (|d_xi x| |d_eta x| |d_zeta x|) at the corner -- the
 *                      quality measure of PAPER.md:1212-1217 (Fig. 7: 0.64); NaN when a
 *                      corner edge has zero length or the hex is NONFINITE; valid over the
 *                      whole input range (|x| <= 2^300: extreme edge scales are evaluated in
 *                      a power-of-two rescaled frame, the measure being scale invariant);
 *   test1_out_opt[i]   1 iff det J > 0 at all 8 corners (Ushakova's Test 1, the 8 corner
 *                      tetrahedra: a necessary condition only, PAPER.md:107-109,
 *                      1260-1263), each sign exact: a corner sample within its fp64
 *                      rounding bound of 0 is re-decided in exact arithmetic (the
 *                      coincident-node rule, then the long accumulator of Step 2), so
 *                      a corner det J that is exactly 0 fails the test.
 * Asynchronous on `stream`; returns HEXVAL_OK or a negative status.              */
int hexval_corner_quality_soa(const double* coords, int64_t n, double* sj_min_out_opt,
                              uint8_t* test1_out_opt, cudaStream_t stream);
int hexval_corner_quality_indexed(const double* vertices, const int32_t* hex_idx, int64_t n,
                                  double* sj_min_out_opt, uint8_t* test1_out_opt,
                                  cudaStream_t stream);

/* Validity and the screening outputs in ONE pass over the coordinates (SURVEY
 * 8(f) NEXT-2 "fused screening outputs"): flags_out exactly as
 * hexval_check_soa / hexval_check_indexed (section 6), and
 * sj_min_out[i] / test1_out[i] exactly as hexval_corner_quality_* (bit-identical:
 * the same corner samples and the same arithmetic), computed by the pass-1
 * kernel from the corner samples it evaluates anyway.  All three outputs are
 * required (device memory); no coefficient output.  Asynchronous on `stream`;
 * returns HEXVAL_OK or a negative status.                                        */
int hexval_check_screen_soa(const double* coords, int64_t n, uint8_t* flags_out,
                            double* sj_min_out, uint8_t* test1_out, cudaStream_t stream);
int hexval_check_screen_indexed(const double* vertices, const int32_t* hex_idx, int64_t n,
                                uint8_t* flags_out, double* sj_min_out, uint8_t* test1_out,
                                cudaStream_t stream);

/* ---- NEXT-1: certified bounds on min det J ------------------------------------
 * For every hex: lower_out[i] <= min over [0,1]^3 of det J <= upper_out[i] (device
 * memory, n doubles each).  lower = min of the Bezier coefficients over the leaves of
 * a subdivision tree (convex hull property), upper = min of the
 * corner coefficients met (actual values); the bounds are
 * "sharpened ... by subdividing": a subdomain is split while the
 * min of its coefficients is < upper - tol, tol = rel_tol * max|b_root| (DESIGN.md
 * reading G15), depth cap HEXVAL_MAX_DEPTH.  On return upper - lower <= tol unless
 * status bit 0 (depth cap reached) is set.  status_out_opt (n bytes, may be NULL):
 * bit 0 capped, bit 1 NONFINITE (then both bounds are NaN).  nodes_dev_opt: NULL or a
 * device counter to which the number of split subdomains is added.
 * rel_tol >= 0 (else HEXVAL_ERR_ARGUMENT).  Asynchronous on `stream`.           */
int hexval_min_detj_bounds_soa(const double* coords, int64_t n, double rel_tol,
                               double* lower_out, double* upper_out, uint8_t* status_out_opt,
                               unsigned long long* nodes_dev_opt, cudaStream_t stream);
int hexval_min_detj_bounds_indexed(const double* vertices, const int32_t* hex_idx, int64_t n,
                                   double rel_tol, double* lower_out, double* upper_out,
                                   uint8_t* status_out_opt, unsigned long long* nodes_dev_opt,
                                   cudaStream_t stream);

/* ---- NEXT-3: candidate-set filtering (indirect hex meshing) -------------------
 * The paper's motivating workload checks candidate hexahedra built from a tet mesh
 * and keeps the valid ones.  From a flags array (n
 * bytes, as written by the calls above):
 *   ids_out_opt       NULL or n int32: the ids i with (flags[i] & 3) == VALID in
 *                     increasing order (the first *count_dev entries are written);
 *   count_dev         device long long: number of VALID entries (required);
 *   group_opt         NULL or n int32 group ids in [0, n_groups) (e.g. grid cell of
 *                     candidate i); precondition, not checked;
 *   group_counts_opt  NULL iff group_opt is NULL; n_groups int32 counters to which
 *                     the number of VALID candidates of each group is ADDED (the
 *                     caller zeroes them first).
 * Device memory, asynchronous on `stream`.                                        */
int hexval_select_valid(const uint8_t* flags, int64_t n, const int32_t* group_opt, int64_t n_groups,
                        int32_t* ids_out_opt, long long* count_dev, int32_t* group_counts_opt,
                        cudaStream_t stream);

/* ---- NEXT-4: linear quadrangles (section 2.1) ---------
 * coords      SoA, 8 planes of n doubles: coords[(2*k + a)*n + i] is axis a (x, y) of
 *             node k = 0..3 of quad i, counter-clockwise (shape functions PAPER.md:290-297).
 * flags_out   n bytes: VALID iff det J > 0 at all four corners (det J is bilinear, its
 *             minimum is a corner value), INVALID otherwise (an exact
 *             zero is INVALID, reading G2; values within the fp64 rounding bound of 0
 *             are decided exactly), NONFINITE for a NaN/Inf or |x| > 2^300 coordinate.
 * J_out_opt   NULL or 4*n doubles: J_out[k*n + i] = det J at corner k+1 (J1 = v12 x v14,
 *             J2 = v12 x v23, J3 = v43 x v23, J4 = v43 x v14; reading Q1 in DESIGN.md).
 * Device memory, asynchronous on `stream`.                                        */
int hexval_check_quad_soa(const double* coords, int64_t n, uint8_t* flags_out, double* J_out_opt,
                          cudaStream_t stream);

/* ---- host-resident calls (synchronous, end to end) --------------------------
 * Same layouts, but every pointer is HOST memory (pinned memory gives
 * overlapped copies; pageable memory works but serialises).  The library
 * copies the inputs to the device in chunks of chunk_hexes hexes (<= 0 picks
 * a default), runs the device path on each chunk while the next chunk's copy
 * is in flight (two internal streams), copies flags (and coefficients) back
 * and returns after everything has landed in host memory.  `stream` orders
 * the work after prior work on that stream (may be 0).                      */
int hexval_check_soa_host(const double* coords_host, int64_t n, uint8_t* flags_host,
                          double* coeffs_host_opt, int64_t chunk_hexes, cudaStream_t stream);

int hexval_check_indexed_host(const double* vertices_host, int64_t nv,
                              const int32_t* hex_idx_host, int64_t n, uint8_t* flags_host,
                              double* coeffs_host_opt, int64_t chunk_hexes,
                              cudaStream_t stream);

/* ---- profiling ---------------------------------------------------------------
 * create/destroy a profile object; pass it to *_ex; after synchronising the
 * stream, hexval_profile_read() adds up the elapsed time of every recorded
 * phase since the last read into ms_out[HEXVAL_NUM_PHASES] and the launch
 * counts into launches_out[HEXVAL_NUM_PHASES] (either may be NULL), then
 * resets.  Returns HEXVAL_OK or HEXVAL_ERR_CUDA.  A profile records at most
 * 256 calls between reads; a *_ex call with a full profile returns
 * HEXVAL_ERR_ARGUMENT and launches nothing.  Each phase is bracketed by a CUDA
 * event pair on the call's stream, which adds a launch bubble to the recorded
 * time.                                          */
hexval_profile* hexval_profile_create(void);
void hexval_profile_destroy(hexval_profile* p);
int hexval_profile_read(hexval_profile* p, double* ms_out, long long* launches_out);

/* ---- scratch ----------------------------------------------------------------
 * The library owns a memory pool per device (cudaMemPoolCreate; the process's
 * default pool is not modified) and persistent scratch arenas carved from it:
 * a call borrows the arena its stream used last, else an arena whose last use
 * has completed, else a new one (arenas = streams with calls in flight at the
 * same time).  An arena holds a 256-B control block, two int32 queues of n
 * entries and the subdivision kernel's node stacks (~1.1 MB per resident warp,
 * the depth-sorted stack's worst case); it grows only when a call needs more.
 * Calls enqueued during CUDA-graph capture allocate from the pool per call
 * instead (graph memory nodes).
 * hexval_scratch_info: bytes reserved by the arenas of `device` and their
 *   number (either output may be NULL).  Host-only; no CUDA call.
 * hexval_scratch_release: frees every idle arena of the current device (waits
 *   for their last uses) and trims the pool.  Returns HEXVAL_OK or
 *   HEXVAL_ERR_CUDA.                                                          */
int hexval_scratch_info(int device, size_t* bytes_reserved_out, int* arenas_out);
int hexval_scratch_release(void);

/* ---- roofline probe (diag.cu; not the hot path) --------------------------
 * Measured FP64 pipe throughput of the current device, the denominator of the
 * FP64 rooflines (the subdivision kernel and indexed pass 1 are
 * FP64 bound): a DFMA-only kernel (8 independent chains per thread, 8 x 256
 * threads per SM, `iters` iterations, best of 5 timed launches on `stream`).
 * *dfma_per_s_out = DFMA lane-instructions per second (1 DFMA = 2 flops);
 * *best_ms_out (optional) = the best launch time.  Synchronises `stream`.
 * Returns HEXVAL_OK, HEXVAL_ERR_ARGUMENT (iters <= 0 or NULL output),
 * HEXVAL_ERR_ALLOC or HEXVAL_ERR_CUDA.                                      */
int hexval_diag_fp64_peak(int iters, double* dfma_per_s_out, float* best_ms_out, cudaStream_t stream);

/* ---- misc -------------------------------------------------------------- */
const char* hexval_status_string(int status);
int hexval_version(void);              /* 100 * major + minor                */
int hexval_kernel_launches_per_call(void); /* kernels one device call enqueues */

#ifdef __cplusplus
}
#endif
#endif /* HEXVAL_H */
