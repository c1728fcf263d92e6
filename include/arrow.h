/* include/arrow.h -- C ABI of the B200 arrow-decomposition SpMM library (libarrow_b200.so).
 *
 * The one operation: Y = A X for a sparse n x n matrix A with a symmetric pattern and a
 * tall-skinny dense X (n x k), evaluated through an arrow matrix decomposition
 *
 *     A X = sum_i P_{pi_i} ( B_i ( P_{pi_i}^T X ) )                    PAPER.md Eq. (1)
 *
 * where every B_i has arrow-width b: nonzeros only in the first b rows/columns or in
 * the b x b diagonal tiles (block-diagonal band of §4.1).  The
 * decomposition (LA-Decompose with random-spanning-forest arrangements, §5.1/§5.3/
 * §5.4) is host preprocessing done once in arrow_plan_create; arrow_spmm is
 * the per-iteration hot path (the paper's setting T >> 1) and runs entirely in
 * hand-written sm_100a CUDA kernels on the caller's stream.  There is no CPU fallback:
 * without a usable CUDA device every call that needs one returns ARROW_E_CUDA.
 *
 * Conventions (all entry points):
 *   - Every call returns arrow_status; nothing throws or aborts across the boundary.
 *     A human-readable detail of the last failure on this thread: arrow_last_error().
 *   - Host inputs are borrowed for the duration of the call and deep-copied.
 *   - A plan owns all its device memory; it is bound to the device current at creation.
 *   - Numbering is 0-based; positions [0, b) of every level are its head (R2).
 *
 * Readings of the paper used by the boundary are listed in DESIGN.md §3 (R1-R23).
 */
#ifndef ARROW_B200_H
#define ARROW_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ARROW_ABI_VERSION 1

typedef enum {
    ARROW_OK = 0,
    ARROW_E_INVALID_ARG = 1,    /* null pointer, b < 2, levels < 0, k < 0, bad dtype/option, aliasing */
    ARROW_E_BAD_CSR = 2,        /* row_ptr not 0-based/nondecreasing, col out of [0,n), unsorted or duplicate columns */
    ARROW_E_NOT_SYMMETRIC = 3,  /* pattern of A is not symmetric (§2: undirected G) */
    ARROW_E_LEVELS = 4,         /* `levels` cap reached with entries left and residual mode is ERROR */
    ARROW_E_CUDA = 5,           /* no device / launch / allocation / asynchronous CUDA error; plan unusable */
    ARROW_E_NCCL = 6,           /* NCCL failure (distributed mode) */
    ARROW_E_NOMEM = 7,          /* host allocation failed */
    ARROW_E_STATE = 8,          /* wrong device current, plan poisoned, collective misuse */
    ARROW_E_UNSUPPORTED = 9     /* size beyond the implementation's index widths, feature not built */
} arrow_status;

typedef enum { ARROW_DTYPE_DEFAULT = -1,  /* options.compute only: same as A's dtype */
               ARROW_F32 = 0, ARROW_F64 = 1 } arrow_dtype;

/* Canonical CSR of A, host memory, borrowed.  row_ptr[0] = 0, nondecreasing,
 * row_ptr[n] = nnz; col_idx in [0, n), strictly increasing within each row (no
 * duplicates); values[nnz] of `dtype`.  Self-loops are allowed (they land in the head
 * or their diagonal tile, R21).  The PATTERN must be symmetric; values need not be. */
typedef struct {
    int64_t n;
    int64_t nnz;
    const int64_t *row_ptr;     /* [n + 1] */
    const int32_t *col_idx;     /* [nnz]   */
    const void *values;         /* [nnz] of dtype */
    arrow_dtype dtype;
} arrow_csr;

typedef struct arrow_plan_s *arrow_plan;
typedef struct arrow_comm_s *arrow_comm;

enum { ARROW_ORDER_ORIGINAL = 0,   /* X, Y rows in A's vertex order (default; R18) */
       ARROW_ORDER_PERMUTED = 1 }; /* X, Y rows in pi_0 order: row p holds vertex perm_0[p] */
/* Step 3 of LA-Decompose: which band around the diagonal a level captures besides the
 * first b rows/columns.  BLOCK: the diagonal b x b tiles (the block-diagonal band Alg. 1 computes,
 * §4.1; reading R3, default).  STRICT: every entry with |p - q| <= b -- the arrow-width
 * definition itself and Fig. 3; fewer levels, body rows read X rows of the
 * neighbouring tiles.  Distributed plans fetch those rows from the ranks that own
 * them: level 0 next to the head block D0 (before level 0 runs), levels >= 1 with the forward rows. */
enum { ARROW_BAND_BLOCK = 0, ARROW_BAND_STRICT = 1 };
enum { ARROW_RESIDUAL_ERROR = 0,   /* levels cap hit with entries left -> ARROW_E_LEVELS */
       ARROW_RESIDUAL_CSR = 1 };   /* keep the leftover entries as one unstructured CSR level */

typedef struct {
    arrow_dtype compute;        /* element type of X, Y and the stored values; default = A's dtype.
                                   fp64 -> fp32 conversion of values rounds to nearest. */
    uint64_t seed;              /* s_decomp of the random spanning forests (R9); default 4 */
    int32_t order;              /* ARROW_ORDER_*; default ORIGINAL.  Distributed mode forces PERMUTED. */
    int32_t residual;           /* ARROW_RESIDUAL_*; default ERROR */
    int64_t window_rows;        /* tile-window (rows) ordering the work for L2 reuse; 0 = default (single GPU:
                                   65536 for level 0, 16384 for levels >= 1; distributed: 16384); rows of
                                   <= 128 bytes run faster with 65536 everywhere */
    int32_t head_chunk;         /* max entries per head-row work segment; 0 = default (32; 128 with
                                   ARROW_FLAG_DETERMINISTIC, one slot per segment) */
    int32_t batch_segments;     /* segments per K-A work batch of full-warp rows: 0 = default = 16 (the only
                                   value accepted; short rows are taken 32 at a time) */
    int32_t band;               /* ARROW_BAND_*: step 3's band; default BLOCK */
    int32_t flags;              /* ARROW_FLAG_* bits; default 0 */
    int32_t transport;          /* ARROW_TRANSPORT_* (distributed plans); default AUTO */
    int32_t home_levels;        /* ARROW_FLAG_HOME_AWARE: levels 1..home_levels home-set-aware; 0 = default
                                   (1 for 2 ranks, 3 for more; measured) */
    int32_t reserved[2];
} arrow_options;

/* options.flags */
enum { ARROW_FLAG_NO_GRAPHS = 1,       /* single GPU: launch the kernels of each call directly instead of
                                          replaying one CUDA graph per (X, Y, k, stream) */
       ARROW_FLAG_DETERMINISTIC = 2,   /* single GPU: bitwise reproducible results -- the head-row partials of
                                          each tile window are stored into their own slots and added in a
                                          fixed order by a per-level epilogue (K-C, Alg. 1 line 3) instead of
                                          L2 atomics (costs time: DESIGN.md §7) */
       ARROW_FLAG_GPU_DECOMPOSE = 4,   /* arrow_plan_create_ex: run LA-Decompose on the current CUDA device
                                          (arrow_decompose_gpu) instead of the host; same decomposition */
       ARROW_FLAG_HOME_AWARE = 8,      /* arrow_plan_create_ex with a comm: home-set-aware arrangement for the
                                          comm's ranks (arrow_decompose_homes, homes = nranks, home_levels =
                                          options.home_levels) */
       ARROW_FLAGS_ALL = 15 };
/* options.transport (distributed plans): AUTO = P2P when every peer's memory can be mapped (CUDA IPC
 * over NVLink), else NCCL; P2P fails with ARROW_E_UNSUPPORTED if a peer cannot be mapped. */
enum { ARROW_TRANSPORT_AUTO = 0, ARROW_TRANSPORT_P2P = 1, ARROW_TRANSPORT_NCCL = 2 };

/* Fill *opt with the defaults above (compute = ARROW_F32 until a CSR is seen: callers that
 * want "same as A" leave compute = -1 after this call, which is what the default sets). */
arrow_status arrow_options_default(arrow_options *opt);

typedef struct arrow_decomposition_s *arrow_decomposition;

/* ---------------------------------------------------------------- north-star trio */

/* Decompose A (LA-Decompose; pruning P:809; random MSF arrangement P:887-896;
 * smallest-first tree order P:900/P:931; block-diagonal extraction P:467/P:473) with arrow
 * width b >= 2 and at most `levels` arrow matrices (0 = no cap: loop until the remainder is
 * empty, R7), then build and upload the device layout.  Validation order: arguments,
 * canonical CSR, pattern symmetry, decomposition, device allocation.  On any error *out is
 * set to NULL and nothing leaks.  The plan binds to the current CUDA device. */
arrow_status arrow_plan_create(const arrow_csr *A, int64_t b, int32_t levels, arrow_plan *out);

/* Y = A X.  X, Y: DEVICE pointers on the plan's device, row-major n x k (leading dimension k),
 * of the plan's dtype, not overlapping (ARROW_E_INVALID_ARG).  Y is fully overwritten
 * (zero rows included).  Stream-ordered on the plan's stream (default: the legacy default
 * stream; see arrow_plan_set_stream); returns after enqueue.  Asynchronous faults surface at
 * the caller's next synchronisation and poison the plan (ARROW_E_CUDA).  k = 0 is a no-op.
 * Workspaces are sized for the largest k seen; call arrow_plan_reserve before graph capture. */
arrow_status arrow_spmm(arrow_plan plan, const void *X, void *Y, int64_t k);

/* Synchronises the plan's device work, frees everything.  NULL is a no-op.  For a distributed plan
 * of the P2P transport the call is COLLECTIVE (every rank must call it, before arrow_comm_destroy):
 * peers read each other's workspaces, so no rank frees its own until all have drained. */
arrow_status arrow_plan_destroy(arrow_plan plan);

/* ---------------------------------------------------------------- extended */

/* As arrow_plan_create with options; comm != NULL selects distributed mode (one process per
 * GPU, every rank passes the same A, b, levels and options; see arrow_comm_create). */
arrow_status arrow_plan_create_ex(const arrow_csr *A, int64_t b, int32_t levels,
                                  const arrow_options *opt, arrow_comm comm, arrow_plan *out);

/* `stream` is a cudaStream_t (NULL = legacy default stream). */
arrow_status arrow_plan_set_stream(arrow_plan plan, void *stream);

/* arrow_spmm on an explicit stream. */
arrow_status arrow_spmm_ex(arrow_plan plan, const void *X, void *Y, int64_t k, void *stream);

/* End-to-end call with HOST buffers: copies X (n x k, plan dtype; pinned memory recommended)
 * to the device, runs arrow_spmm, copies Y back, and synchronises `stream` before returning.
 * Device staging buffers are owned by the plan and reused. */
arrow_status arrow_spmm_host(arrow_plan plan, const void *X_host, void *Y_host, int64_t k, void *stream);

/* Batched end-to-end call: Y_host[c] = A X_host[c] for c = 0..count-1, each an n x k HOST buffer
 * of the plan's dtype (pinned memory needed for the overlap), e.g. several feature matrices
 * multiplied by the same A (preprocessing amortised over many products).  The copies are
 * pipelined with the kernels through two device slots owned by the plan: the H2D copy of X[c+1]
 * and the D2H copy of Y[c-1] run on two copy streams while the kernels of c run on `stream` (PCIe
 * is full duplex).  Distributed plans: every rank passes its local rows (n_local x k) and the same
 * count (collective, like arrow_spmm).  Synchronises `stream` before returning.  count < 0 or a
 * NULL pointer: ARROW_E_INVALID_ARG. */
arrow_status arrow_spmm_host_batch(arrow_plan plan, const void *const *X_host, void *const *Y_host,
                                   int64_t count, int64_t k, void *stream);

/* Iterated SpMM with a fused activation (the paper's use case of repeated
 * products with the rows left in pi_0 order):  X_{t+1} = act(A X_t), t = 0..iters-1.
 * X and Y are both n x k device buffers of the plan's dtype (row order of the plan: original,
 * or pi_0 with ARROW_ORDER_PERMUTED) and are used as a ping-pong pair: X holds X_0 on entry and
 * both are overwritten; *result_in_y (may be NULL) is set to 1 if X_iters ends in Y (iters odd),
 * 0 if it ends in X.  activation: ARROW_ACT_NONE or ARROW_ACT_RELU.  The activation is applied
 * inside K-A when a row's last segment is flushed (kFinalBit, computed at plan time); rows last
 * written by head-row partials get one small pass per iteration.  Single-GPU plans only
 * (ARROW_E_UNSUPPORTED for distributed plans); iters < 1 or an unknown activation ->
 * ARROW_E_INVALID_ARG; stream-ordered on `stream` (NULL = legacy default stream). */
enum { ARROW_ACT_NONE = 0, ARROW_ACT_RELU = 1 };
arrow_status arrow_spmm_iterate(arrow_plan plan, void *X, void *Y, int64_t k, int32_t iters, int32_t activation,
                                void *stream, int32_t *result_in_y);

/* Pre-size the k-dependent workspaces (head block D0, head accumulator C0) for k <= k_max so
 * that later arrow_spmm calls allocate nothing (CUDA-graph capture safe). */
arrow_status arrow_plan_reserve(arrow_plan plan, int64_t k_max);

typedef struct {
    int64_t n, nnz, b;
    int32_t levels;             /* number of arrow matrices (order of the decomposition) */
    int32_t dtype;              /* arrow_dtype */
    int32_t order;              /* ARROW_ORDER_* */
    int32_t distributed;        /* 1 if built with a comm */
    int64_t residual_nnz;       /* entries in the residual CSR level (0 unless RESIDUAL_CSR) */
    int64_t sum_rows;           /* sum_i n_i */
    int64_t isolated;           /* vertices with no entry in A (level-0 zero rows) */
    double create_seconds;      /* wall time of decomposition + layout build + upload */
    /* algorithmic bytes per SpMM (from the [iffalse] IO lemma P:1061-1066):
     *   B_alg(k) = bytes_alg_fixed + bytes_alg_rows * k * sizeof(dtype)                      */
    int64_t bytes_alg_fixed;    /* sum_i nnz_i (s+4) + (rows_i+1) 8 + rows_i 4 */
    int64_t bytes_alg_rows;     /* sum_i cols_i + n + sum_{i>=1} 2 n_i  (rows moved per unit k*s) */
    int64_t device_bytes;       /* device memory held by the plan (excluding k workspaces) */
    int64_t reserved[8];
} arrow_plan_info_t;

arrow_status arrow_plan_info(arrow_plan plan, arrow_plan_info_t *info);

typedef struct {
    int64_t rows;               /* n for level 0 (A-isolated vertices appended as empty rows), n_i otherwise */
    int64_t n_i;                /* vertices with an entry in A_i (R8) */
    int64_t head;               /* h_i = min(b, n_i) */
    int64_t nnz;                /* entries of B_i */
    int64_t head_nnz;           /* entries in the head rows [0, h_i) */
    int64_t tiles;              /* ceil(n_i / b) */
    int64_t segments;           /* device work segments of this level */
    int64_t reserved[4];
} arrow_level_info_t;

arrow_status arrow_plan_level_info(arrow_plan plan, int32_t level, arrow_level_info_t *info);

/* Canonical B_i in positions (for bit-exact structure parity): perm[rows] = original vertex at
 * each position (pi_i^{-1}), row_ptr[rows+1], col[nnz] positions sorted within each row,
 * val[nnz] of the plan's dtype.  Any output pointer may be NULL to skip it.  Host memory. */
arrow_status arrow_plan_export_level(arrow_plan plan, int32_t level, int32_t *perm, int64_t *row_ptr,
                                     int32_t *col, void *val);

/* Distributed mode: this rank's contiguous pi_0-order row range [begin, end) of X and Y. */
arrow_status arrow_plan_local_rows(arrow_plan plan, int64_t *begin, int64_t *end);

/* Per-kernel device time accumulated with CUDA events on the launching stream while profiling
 * is on (arrow_plan_set_profiling).  Index by arrow_kernel_id. */
enum { ARROW_K_HEAD_STAGE = 0,  /* S0: D0 = X[head], C0 = 0 */
       ARROW_K_SEGMENTS = 1,    /* S1+S2: body rows and head slices (the dominant kernel) */
       ARROW_K_HEAD_EPI = 2,    /* S3: Y[head] (=|+=) C0 */
       ARROW_K_COMM = 3,        /* S6: NCCL calls + pack/unpack (distributed) */
       ARROW_K_COUNT = 4 };
typedef struct {
    double ms[ARROW_K_COUNT];
    int64_t launches[ARROW_K_COUNT];
    int64_t calls;              /* arrow_spmm calls profiled */
    double launch_ms[16];       /* by position of the launch within a call (first 16 launches) */
} arrow_kernel_times_t;

arrow_status arrow_plan_set_profiling(arrow_plan plan, int32_t on);   /* on: resets the counters */
arrow_status arrow_plan_kernel_times(arrow_plan plan, arrow_kernel_times_t *out); /* synchronises */

/* ---------------------------------------------------------------- host decomposition object
 * The preprocessing half of arrow_plan_create, exposed so that a decomposition can be computed
 * once, checked, saved and shared (every rank of a distributed run can load the same file).
 * Host only -- no CUDA device is needed -- except arrow_decompose_gpu and arrow_decompose_homes with
 * device = 1, which compute on the current device (the result still lives on the host). */

/* LA-Decompose of A (same algorithm and readings as arrow_plan_create).  keep_residual != 0
 * keeps entries left at the `levels` cap instead of failing with ARROW_E_LEVELS. */
arrow_status arrow_decompose(const arrow_csr *A, int64_t b, int32_t levels, uint64_t seed, int32_t keep_residual,
                             arrow_decomposition *out);
/* Same with step 3's band chosen (ARROW_BAND_BLOCK = arrow_decompose, ARROW_BAND_STRICT: |p-q| <= b,
 * P:253 / Fig. 3); any other value -> ARROW_E_INVALID_ARG.  Saved files record the band. */
arrow_status arrow_decompose_ex(const arrow_csr *A, int64_t b, int32_t levels, uint64_t seed, int32_t keep_residual,
                                int32_t band, arrow_decomposition *out);
/* Same as arrow_decompose_ex, computed on the CURRENT CUDA device (§5.1
 * P:805-814 with §5.3 P:887-896 and §5.4): a bit-identical decomposition -- the same
 * degree-ordered heads, the same keyed minimum spanning forests (Boruvka under the strict (key, u, v)
 * order finds the forest Kruskal finds), the same smallest-first tree layout (Euler-tour list ranking
 * in place of the host's DFS).  A is read from HOST memory and the result lives on the host like
 * arrow_decompose's; device scratch is allocated and freed inside the call (the default stream,
 * synchronous).  Errors as arrow_decompose_ex, plus: n >= 2^30 or nnz >= 2^31 - 1 ->
 * ARROW_E_INVALID_ARG; no device, allocation or launch failure -> ARROW_E_CUDA. */
arrow_status arrow_decompose_gpu(const arrow_csr *A, int64_t b, int32_t levels, uint64_t seed, int32_t keep_residual,
                                 int32_t band, arrow_decomposition *out);
/* The general form: homes = G in [1, 8] lays levels >= 1 out for G ranks (reading
 * R25 of DESIGN.md §3; an extension, not in the paper): after level 0 every vertex gets the home range
 * of its pi_0 position -- G contiguous ranges of whole level-0 tiles balanced by level-0 work plus
 * every vertex's entries left for levels >= 1 -- and in the levels 1..home_levels the forest uses only
 * the edges inside one home and its trees are laid out by (home of the root, size desc, min id asc)
 * instead of (size desc, min id asc), so a distributed plan for G
 * ranks computes those levels' home-g trees on rank g and moves few of their rows over NVLink; edges
 * between homes wait for a later level, so more home-aware levels mean more levels and rows
 * (DESIGN.md §8 measures the trade); home_levels = 0 picks the default (1 for homes = 2, else 3).
 * homes = 1 is arrow_decompose_ex (home_levels ignored).  device: 0 = host, 1 = the current CUDA device (as
 * arrow_decompose_gpu; the same decomposition).  Errors as arrow_decompose_ex / _gpu; homes outside
 * [1, 8] or device not 0/1 -> ARROW_E_INVALID_ARG.  Saved files (format 3) record the homes. */
arrow_status arrow_decompose_homes(const arrow_csr *A, int64_t b, int32_t levels, uint64_t seed, int32_t keep_residual,
                                   int32_t band, int32_t homes, int32_t home_levels, int32_t device,
                                   arrow_decomposition *out);
/* homes and home_levels of a decomposition (either pointer may be NULL) and, when homes > 1 and
 * ranges != NULL, level = -1: the pi_0 home ranges ranges[0..homes]; level in 1..home_levels: the
 * first position of each home's trees (ranges[g] .. ranges[g+1] hold home g's trees, ranges[0] = head,
 * ranges[homes] = n_i); any other level -> ARROW_E_INVALID_ARG. */
arrow_status arrow_decomposition_homes(arrow_decomposition d, int32_t level, int32_t *homes, int32_t *home_levels,
                                       int64_t *ranges);
/* n, b, order (number of arrow matrices), residual entries; any pointer may be NULL. */
arrow_status arrow_decomposition_info(arrow_decomposition d, int64_t *n, int64_t *b, int32_t *levels,
                                      int64_t *residual_nnz);
arrow_status arrow_decomposition_level_info(arrow_decomposition d, int32_t level, arrow_level_info_t *info);
/* Canonical B_i in positions (see arrow_plan_export_level); values as fp64 (exact for fp32/fp64 A). */
arrow_status arrow_decomposition_export_level(arrow_decomposition d, int32_t level, int32_t *perm, int64_t *row_ptr,
                                              int32_t *col, double *val);
/* Residual entries (original ids, CSR order): u[r], v[r], val[r]. */
arrow_status arrow_decomposition_export_residual(arrow_decomposition d, int32_t *u, int32_t *v, double *val);
/* Versioned little-endian binary file with a 64-bit FNV-1a checksum; load verifies it. */
arrow_status arrow_decomposition_save(arrow_decomposition d, const char *path);
arrow_status arrow_decomposition_load(const char *path, arrow_decomposition *out);
arrow_status arrow_decomposition_destroy(arrow_decomposition d);
/* Build a device plan from a decomposition (options as arrow_plan_create_ex; opt->seed and the
 * residual mode are taken from the decomposition). */
arrow_status arrow_plan_create_from(arrow_decomposition d, const arrow_options *opt, arrow_comm comm, arrow_plan *out);

/* ---------------------------------------------------------------- distributed (NCCL) */
/* One process per GPU.  Rank 0 calls arrow_comm_unique_id and shares the 128 bytes (e.g.
 * torch.distributed.broadcast_object_list); every rank then calls arrow_comm_create with its
 * device current.  Collectives: per-level broadcast of the head block and reduction of the
 * head partials (Alg. 1), plus the inter-level exchange of moved rows (Alg. 2,
 * P:484-499). */
arrow_status arrow_comm_unique_id(uint8_t id[128]);
arrow_status arrow_comm_create(int32_t nranks, int32_t rank, const uint8_t id[128], arrow_comm *out);
arrow_status arrow_comm_destroy(arrow_comm comm);

/* Host-only view of the distributed schedule of `rank` among `nranks` (no GPU, no NCCL): its pi_0
 * row range lohi[2] = [begin, end) and, if counts != NULL, per arrow level 4*nranks + 4 int64:
 * rows sent to / received from each rank in the forward exchange (X rows its tiles need), rows
 * sent to / received from each rank in the reverse exchange (level>=1 results going home), then
 * entries, segments, head rows owned and zero rows of its local work.  Used to test routing on
 * CPU (what rank a sends to b must equal what b expects from a). */
arrow_status arrow_dist_schedule(arrow_decomposition d, int32_t nranks, int32_t rank, int64_t window_rows,
                                 int32_t head_chunk, int64_t *lohi, int64_t *counts);

/* ---------------------------------------------------------------- diagnostics */
const char *arrow_status_string(arrow_status s);
const char *arrow_last_error(void);          /* thread-local detail of the last failure ("" if none) */
int32_t arrow_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* ARROW_B200_H */
