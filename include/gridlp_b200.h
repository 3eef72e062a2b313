/*
 * gridlp_b200.h — C ABI of libgridlp_b200.so, the sm_100a (B200) kernels for
 * the hot path of arXiv 2601.07628 ("distributed PDHG over a 2D grid
 * partition of A"): FP64 CSR products A·x̄ and Aᵀ·y fused with the
 * restarted-Halpern PDHG update and with the KKT / restart reductions.
 *
 * Every entry point here replaces a call site of the reference package
 * `gridlp` (pure Python; /root/reference/pkg/src/gridlp). The replaced
 * reference interface is cited (file:line) on each declaration.
 *
 * Conventions
 *  - Plain pointers and sizes only; no torch types. All pointers are DEVICE
 *    pointers unless a parameter says "host". The caller (Python/PyTorch)
 *    owns every allocation; the library allocates nothing and keeps no
 *    state except the thread-local error string.
 *  - Every function returns 0 on success or a positive gridlp error code;
 *    gridlp_last_error() returns a description of the last failure on the
 *    calling thread. Launches are asynchronous and stream-ordered
 *    (`stream` is a cudaStream_t passed as void*), so they can be captured
 *    into CUDA graphs.
 *  - Arithmetic is IEEE FP64 with explicit round-to-nearest multiplies and
 *    adds (no FMA contraction), mirroring the reference's numpy/scipy
 *    expressions operation for operation. Row sums are sequential
 *    left-to-right from +0.0 like scipy's csr_matvec for every row of at
 *    most `exact_row_max` entries (bit-identical to the reference); longer
 *    rows use a deterministic tree sum (run-to-run reproducible, FP64
 *    tolerance vs the reference).
 *  - Reductions (norms, dots) are deterministic: per-CTA partials in a fixed
 *    tree order, then one fixed-order final pass.
 */
#ifndef GRIDLP_B200_H
#define GRIDLP_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GRIDLP_ABI_VERSION 2

enum gridlp_status {
  GRIDLP_OK = 0,
  GRIDLP_ERR_ARG = 1,      /* invalid argument (ValueError in the reference) */
  GRIDLP_ERR_CUDA = 2,     /* CUDA launch / runtime failure                   */
  GRIDLP_ERR_WORKSPACE = 3, /* reduction workspace too small                  */
  GRIDLP_ERR_UNSUPPORTED = 4 /* valid input this entry point does not handle (caller falls back) */
};

/* Max number of reduction slots an op can produce (see gridlp_red_t). */
#define GRIDLP_MAX_RED 8
/* Max partial products summed by an unfused epilogue (grid rows/cols). */
#define GRIDLP_MAX_PARTS 16
/* Entries per chunk of a heavy row (one CTA sums one chunk). */
#define GRIDLP_HEAVY_CHUNK 2048
/* Largest light_row_max / exact_row_max accepted. */
#define GRIDLP_ROW_MAX_LIMIT 65536

/* Value storage of a block (gridlp_csr_t.val_codec). Every codec is
 * LOSSLESS: the kernels rebuild the exact FP64 value and multiply it by the
 * gathered entry as with FP64 storage, so products are bit-identical. */
#define GRIDLP_VALS_F64 0   /* sell_vals / long_vals are double (12 B per nonzero)            */
#define GRIDLP_VALS_F32 1   /* ... are float; every value is exactly a float (8 B per nonzero)  */
#define GRIDLP_VALS_UNIT 2  /* every value is +1.0 or -1.0: no value arrays, bit 31 of the
                               column index is the sign (4 B per nonzero; network / MCF rows)   */

/*
 * One device-resident block A_ij (or its stored transpose) in SELL-32 plus
 * a compact CSR of its long rows. Replaces SparseMatrix
 * (lp_model.py:40-150) for a LocalBlock matrix / matrix_transpose
 * (partition.py:93-122): int32 column indices, FP64 values — 12 B/nnz
 * instead of the reference's 16 (8 or 4 B/nnz with the lossless value codecs,
 * val_codec below). Every row is summed in one of three ways:
 *
 * light (length <= light_row_max): SELL-32. Rows are cut into slices of 32
 *   consecutive rows; inside a slice the lanes are ordered by row length
 *   (descending, stable) and entry j of lane l is stored at
 *   sell_*[slice_off[s] + 32 j + l] in the row's original entry order, so a
 *   warp step reads 32 consecutive values and column indices; each lane
 *   adds its row left to right from +0.0 (bit-identical to scipy).
 *   lane_info[32 s + l] = (row length << 8) | (row & 31), or -1 for an empty
 *   lane (long row or past the end).
 * long exact (light_row_max < length <= exact_row_max): compact CSR
 *   long_rows / long_ptr / long_cols / long_vals; exact_long lists the
 *   compact-CSR indices h of these rows. One warp per row computes 32
 *   products per step and adds them to one running sum in entry order
 *   (bit-identical to scipy).
 * heavy (length > exact_row_max): the compact-CSR row h is cut into chunks
 *   of GRIDLP_HEAVY_CHUNK entries, chunk_first[h] .. chunk_first[h+1]-1
 *   (empty for long exact rows), chunk_row[c] = h; one CTA per chunk
 *   tree-sums it and the last-arriving chunk CTA adds the chunk sums in
 *   chunk order (deterministic, FP64 tolerance vs the reference).
 *
 * chunk_sums (one double per chunk) and chunk_done (one int per long row,
 * zero before the first launch, left zero by every launch) are
 * caller-owned scratch; products over the same block must be
 * stream-ordered.
 */
typedef struct gridlp_csr {
  int64_t num_rows;
  int64_t num_cols;
  int64_t nnz;                /* < 2^31 per block (int32 row pointers in the setup); SELL offsets are int64 */
  const double* sell_vals;    /* [slice_off[num_slices]] */
  const int32_t* sell_cols;
  const int64_t* slice_off;   /* [num_slices + 1] (int64: padded SELL entries may pass 2^31) */
  const int32_t* lane_info;   /* [32 * num_slices] */
  int64_t num_slices;         /* ceil(num_rows / 32) */
  const int32_t* long_rows;   /* [num_long_rows] ascending */
  const int32_t* long_ptr;    /* [num_long_rows + 1] */
  const int32_t* long_cols;
  const double* long_vals;
  int64_t num_long_rows;
  const int32_t* exact_long;  /* [num_exact_long] */
  int64_t num_exact_long;
  const int32_t* chunk_first; /* [num_long_rows + 1] */
  const int32_t* chunk_row;   /* [num_chunks] */
  int64_t num_chunks;
  double* chunk_sums;         /* [num_chunks] scratch */
  int32_t* chunk_done;        /* [num_long_rows] scratch, zero-initialised */
  int32_t light_row_max;      /* <= GRIDLP_ROW_MAX_LIMIT */
  int32_t exact_row_max;      /* >= light_row_max, <= GRIDLP_ROW_MAX_LIMIT */
  /* Column bands: a block whose gather vector exceeds L2 may be stored as K
   * CSRs over consecutive column ranges (entries keep their row order, so a
   * row's band-k entries are the next ones of its scipy add chain). Band
   * k > 0 has carry = the row sums of bands < k (written by gridlp_op_store
   * of band k - 1), and every exact row's sequential sum starts from
   * carry[row] instead of 0.0: the result is the unbanded sum bit for bit.
   * Chunked rows (> exact_row_max) must lie wholly in the last band (their
   * carry is then 0 and ignored). NULL = start from 0.0. */
  const double* carry;
  /* Reserved (ignored). Round 2 used it to split the gathers' L2 policy at
   * a hot prefix; measured without gain and removed from the kernels (every
   * gather is L2 evict_last). */
  int64_t hot_cols;
  /* GRIDLP_VALS_*: how sell_vals / long_vals store the values (F32: cast the
   * pointers to const float*; UNIT: both NULL allowed, sell_cols / long_cols
   * carry the sign in bit 31). The setup detects the codec per block from
   * the values themselves (lp_model.py:53-55 stores FP64 values; integer
   * and +-1 coefficients are exact in the narrower forms). */
  int32_t val_codec;
  /* GRIDLP_CSR_* launch hints (never change a value): GRIDLP_CSR_WIDE_CTAS
   * runs the main-loop products' SELL lanes in 4-warp CTAs instead of 2 —
   * fewer CTA launches for blocks of very short rows (network / MCF columns:
   * cfg4's A^T K1 2652 -> 2441 us). */
  int32_t launch_flags;
} gridlp_csr_t;
#define GRIDLP_CSR_WIDE_CTAS 1

/*
 * Peer-memory exchange of one grid axis group (G ranks: a grid row for the
 * C axis, a grid column for the R axis) — the fused replacement of
 * "partial product -> allreduce -> epilogue" (comm.py:322-329). Every rank
 * owns a receive buffer of 2 x G slots of `len` doubles and an arrival
 * counter, mapped into all group members (CUDA IPC; NVLink P2P across
 * GPUs). The product kernel writes its partial row sums straight into slot
 * my_slot of every member's buffer (parity = *epoch & 1) and its last CTA
 * signals every member's counter; the consuming epilogue waits until its
 * counter reaches (*epoch + 1) * G, adds the G slots in ascending order —
 * the reference's reduction order, for any G — and the exchange ends with
 * *epoch += 1. Two parities suffice: a rank cannot produce exchange e + 2
 * before every member has produced e + 1, i.e. has consumed e.
 */
typedef struct gridlp_peer {
  double* dst[GRIDLP_MAX_PARTS];     /* receive buffer base of each member */
  uint32_t* flag[GRIDLP_MAX_PARTS];  /* arrival counter of each member */
  double* recv;                      /* this rank's own receive buffer */
  uint32_t* my_flag;                 /* this rank's own arrival counter */
  uint32_t* epoch;                   /* exchanges completed on this axis (device) */
  uint32_t* cta_count;               /* CTAs of the current product done (device scratch, zero) */
  int32_t group_size;
  int32_t my_slot;
  int64_t len;
  int64_t timeout_ns;                /* consumer wait bound (collective_timeout_seconds); 0 = 120 s */
} gridlp_peer_t;

/*
 * Source of the per-row sums an op consumes: either a product with a
 * matrix block (A != NULL: sum_r = (A · gather)_r), or an ascending-order
 * sum of partial vectors (A == NULL: sum_r = ((parts[0]_r + parts[1]_r) +
 * ...), the reduction order of the reference communicator, comm.py:75-84;
 * nparts == 1 after an NCCL allreduce; nparts == 0 means all-zero sums), or
 * (peer != NULL, A == NULL) the G slots of a peer exchange, in slot order.
 */
typedef struct gridlp_src {
  const gridlp_csr_t* A;
  const double* gather;
  const double* parts[GRIDLP_MAX_PARTS];
  int32_t nparts;
  int32_t reserved;
  int64_t num_rows;         /* rows when A == NULL */
  const gridlp_peer_t* peer;
} gridlp_src_t;

/* Step parameters, DEVICE-resident so captured graphs pick up updates.
 * tau = eta/omega, sigma = eta*omega (pdhg_engine.py:61-67); the Halpern
 * counter of an op launched with `iter` is inner_k + iter
 * (pdhg_engine.py:184-189, :396-400). */
typedef struct gridlp_step {
  double tau;
  double sigma;
  double gamma;
  int64_t inner_k;
} gridlp_step_t;

/* Primal-side vectors of one grid column j (length n). x_bar is written by
 * the primal op and gathered by the dual op. */
typedef struct gridlp_primal {
  double* x;
  double* x_bar;
  double* x_anchor;
  const double* c;
  const double* lo;
  const double* hi;
  int64_t n;
  /* Column scale Dc of a diagonally scaled LP (scaling.py: A~ = Dr A Dc,
   * x = Dc x~), NULL when unscaled. When set, gridlp_op_kkt_cols evaluates
   * the KKT terms of the ORIGINAL LP at x = Dc x~ (the restart terms stay
   * in the scaled space); every other op ignores it. */
  const double* scale;
} gridlp_primal_t;

/* Dual-side vectors of one grid row i (length m). */
typedef struct gridlp_dual {
  double* y;
  double* y_anchor;
  const double* lo;   /* con_lower */
  const double* hi;   /* con_upper */
  int64_t m;
  /* Row scale Dr (y = Dr y~), NULL when unscaled: gridlp_op_kkt_rows then
   * reports the original LP's range violation and bound penalty. */
  const double* scale;
} gridlp_dual_t;

/* Reduction workspace: `partials` holds capacity * GRIDLP_MAX_RED doubles;
 * the op writes its final sums to out[0..k). With `terms` (>= rows * k
 * doubles) a fused product stores each row's k reduction terms and they are
 * summed in a fixed row order (the partial-sum path's order): the sums no
 * longer depend on the block's layout (row classes, light_row_max, column
 * bands). terms = NULL: per-CTA partials in layout order. */
typedef struct gridlp_red {
  double* partials;
  int64_t capacity;
  double* out;
  double* terms;
  int64_t terms_capacity;
} gridlp_red_t;

/* flags */
#define GRIDLP_F_HALPERN 1u   /* EngineConfig.halpern (pdhg_engine.py:396-399) */
#define GRIDLP_F_SUMSQ 2u     /* op_store: also reduce sum of squares */
#define GRIDLP_F_STREAM 4u    /* op_store: streaming (evict-first) output, e.g. column-band carries */
#define GRIDLP_F_UNIFORM_BOUNDS 8u /* op_primal / pdhg_iterate: every variable's bounds equal lo[0], hi[0]
                                    * (the arrays stay full length; the op reads two scalars instead) */

/* --- library / device ---------------------------------------------------- */
int gridlp_abi_version(void);
/* Build variant: GRIDLP_BUILD_CHECKED set in the bounds-checked test build
 * (-DGRIDLP_CHECKED: gather indices, SELL lane extents, long-row ranges and
 * written rows verified in the kernels, trap on violation); 0 otherwise. */
#define GRIDLP_BUILD_CHECKED 1
int gridlp_build_flags(void);
const char* gridlp_last_error(void);
/* SM count and L2 size of `device` (host ints). */
int gridlp_device_info(int device, int32_t* sm_count, int64_t* l2_bytes);
/* Let kernels on the current device read and write memory of peer_device
 * (NVLink P2P for the peer exchange); already-enabled is success. */
int gridlp_enable_peer_access(int peer_device);
/* Upper bound on the CTAs (reduction slots) an op over `src` launches. */
int64_t gridlp_op_slots(const gridlp_src_t* src);
/* Process-wide kernel knobs (no reference counterpart; results are
 * bit-identical for every value — they pick kernels, not arithmetic):
 *   "sell_variant"    1 = SELL lanes with the column/value streams issued
 *                     one step block ahead of the gathers (default),
 *                     0 = the round-1 kernel (streams, then gathers)
 *   "chain_products"  gridlp_pdhg_iterate chains its products by
 *                     programmatic dependent launch (default 1)
 * Unknown key or out-of-range value: GRIDLP_ERR_ARG. get returns -1 for an
 * unknown key. */
int gridlp_set_tuning(const char* key, int64_t value);
int64_t gridlp_get_tuning(const char* key);

/* --- products ------------------------------------------------------------ */
/* out = sums(src). Replaces spmv (sparse_kernels.py:18-24) and
 * spmv_transpose (:39-45) when src->A is set, and the vector AllReduce's
 * ascending reduction (comm.py:75-84, :322-329) when src->parts is used.
 * With GRIDLP_F_SUMSQ also red->out[0] = sum of out_r^2 (the power
 * iteration's u_sq / s_sq, sparse_kernels.py:83, :89). */
int gridlp_op_store(const gridlp_src_t* src, double* out, uint32_t flags,
                    const gridlp_red_t* red, void* stream);

/* Product half of a peer exchange: rows of src->A · src->gather written to
 * slot peer->my_slot (current parity) of every group member's receive
 * buffer (and to local_out when not NULL: the block-local partial the
 * fixed-point cross term needs, pdhg_engine.py:257, :426); the product's
 * last CTA signals every member. */
int gridlp_op_store_peer(const gridlp_src_t* src, const gridlp_peer_t* peer, double* local_out, void* stream);

/* --- PDHG iteration halves ------------------------------------------------ */
/* Primal half over grid column j, rows = variables, sums = [Aᵀ y]_j:
 *   x̂ = clip(x - tau (c - aty), lo, hi)             pdhg_engine.py:171-173
 *   x_bar = 2 x̂ - x                                 pdhg_engine.py:233
 *   x <- (w x̂ - gamma x) + x_anchor/(k+2)            pdhg_engine.py:184-189
 * Replaces primal_step + the primal part of halpern_step
 * (pdhg_engine.py:223-228, :238-242; solver_driver.py:376-382). */
int gridlp_op_primal(const gridlp_src_t* src, const gridlp_primal_t* pv,
                     const gridlp_step_t* d_step, int32_t iter, uint32_t flags,
                     void* stream);

/* Dual half over grid row i, rows = constraints, sums = z = [A x̄]_i:
 *   v = y/sigma - z;  ŷ = sigma (v - clip(v, -hi, -lo))   pdhg_engine.py:176-181
 *   y <- (w ŷ - gamma y) + y_anchor/(k+2)
 * Replaces dual_step + the dual part of halpern_step
 * (pdhg_engine.py:231-242; solver_driver.py:378-383). */
int gridlp_op_dual(const gridlp_src_t* src, const gridlp_dual_t* dv,
                   const gridlp_step_t* d_step, int32_t iter, uint32_t flags,
                   void* stream);

/* n_iters PDHG iterations of a block whose axes are not split (R = C = 1,
 * or the single block of a 1x1 grid): per iteration the primal half over
 * primal_src (= Aᵀ y) then the dual half over dual_src (= A x̄), Halpern
 * counter inner_k + t, then inner_k += n_iters on the device. The loop body
 * of iterate_epoch (pdhg_engine.py:394-400; solver_driver.py:376-383); the
 * engine captures the same sequence in a CUDA graph. */
int gridlp_pdhg_iterate(const gridlp_src_t* primal_src, const gridlp_primal_t* pv,
                        const gridlp_src_t* dual_src, const gridlp_dual_t* dv, gridlp_step_t* d_step,
                        int32_t n_iters, uint32_t flags, void* stream);

/* --- KKT pass (pdhg_engine.py:310-346; solver_driver.py:335-358) -------- */
/* Constraint side, sums = [A x]_i. Writes ax (may be NULL) and reduces
 *   out[0] = ||range_violation(ax)||^2            pdhg_engine.py:206-208, :320-321
 *   out[1] = sum over finite hi of hi * max(-y,0)  (bound_penalty(-y), :192-203)
 *   out[2] = sum over finite lo of lo * max(y,0)
 *   out[3] = count of infinite-bound violations (penalty = +inf if > 0). */
int gridlp_op_kkt_rows(const gridlp_src_t* src, const gridlp_dual_t* dv,
                       double* ax, const gridlp_red_t* red, void* stream);

/* Variable side, sums = [Aᵀ y]_j. Writes x_probe_bar = 2 x_probe - x
 * (restart probe input, pdhg_engine.py:420) and reduces
 *   out[0] = ||(x_probe - x)/tau||^2   out[1] = c·x
 *   out[2] = ((x_probe - shifted)/tau)·x   out[3] = ||x - x_probe||^2
 * (pdhg_engine.py:324-336, :424, :255). */
int gridlp_op_kkt_cols(const gridlp_src_t* src, const gridlp_primal_t* pv,
                       double* x_probe_bar, const gridlp_step_t* d_step,
                       const gridlp_red_t* red, void* stream);

/* Restart probe, sums = z_probe = [A x_probe_bar]_i:
 *   y_probe = dual_update(y, z_probe)  dy = y - y_probe
 *   out[0] = ||dy||^2
 *   out[1] = sum 0.5 (ax - z_probe)_r dy_r   (only when ax != NULL; the
 *            fused single-block form of the cross term, pdhg_engine.py:426)
 * dy_out (may be NULL) receives dy for the grid form of the cross term.
 * (pdhg_engine.py:419-427, :245-259; solver_driver.py:403-413). */
int gridlp_op_probe(const gridlp_src_t* src, const gridlp_dual_t* dv,
                    const double* ax, double* dy_out, const gridlp_step_t* d_step,
                    const gridlp_red_t* red, void* stream);

/* out[0] = sum_r 0.5 (a_r - b_r) d_r — the per-block cross term
 * <A_ij dx_j, dy_i> from block-local partial products (pdhg_engine.py:257,
 * :426). */
int gridlp_op_halfdiff_dot(const double* a, const double* b, const double* d,
                           int64_t n, const gridlp_red_t* red, void* stream);

/* out[0] = ||v - anchor||^2 then anchor <- v (restart application:
 * anchor distances pdhg_engine.py:433-442 and anchor reset :448-449). */
int gridlp_op_anchor(double* v, double* anchor, int64_t n,
                     const gridlp_red_t* red, void* stream);

/* out[0] = a·b (power iteration v_sq, sparse_kernels.py:84). */
int gridlp_op_dot(const double* a, const double* b, int64_t n,
                  const gridlp_red_t* red, void* stream);

/* out_r = in_r / divisor (v = s / sqrt(s_sq), sparse_kernels.py:92). */
int gridlp_op_div(const double* in, double* out, int64_t n, double divisor,
                  void* stream);

/* out_r = in_r / sqrt(*sumsq), the divisor read on the device from a
 * reduction slot (the same correctly rounded sqrt and division as
 * gridlp_op_div with divisor = sqrt(s_sq) computed on the host), so a
 * single-block power iteration needs no host round trip per step. */
int gridlp_op_div_norm(const double* in, double* out, int64_t n, const double* sumsq,
                       void* stream);

/* out_r = lo/hi projection of 0 (initial_device_state, pdhg_engine.py:349-353),
 * anchor_r = out_r. */
int gridlp_op_init_primal(const gridlp_primal_t* pv, void* stream);

/* d_step->inner_k += delta on the device (a captured chunk of `delta`
 * iterations advances the Halpern counter itself, pdhg_engine.py:400). */
int gridlp_op_step_advance(gridlp_step_t* d_step, int64_t delta, void* stream);

/* n_iters fused iterations of a single-block grid in ONE cooperative launch
 * (launch-bound LPs, e.g. BASELINE configs[0]): grid-wide barriers between
 * the primal and dual products instead of kernel boundaries; iterates are
 * gridlp_pdhg_iterate's bit for bit. `scratch`: caller-owned device memory of
 * gridlp_persistent_scratch_bytes(), zeroed once before first use (a grid
 * barrier's counter; it resets itself). GRIDLP_ERR_UNSUPPORTED when a matrix
 * has heavy (chunked) rows — use gridlp_pdhg_iterate. Same call site as
 * gridlp_pdhg_iterate (pdhg_engine.py:394-400). */
/* gridlp_pdhg_iterate of n_iters iterations recorded ONCE as a CUDA graph
 * (stream capture on a private stream, no synchronisation, so the device
 * keeps running earlier work while the host captures and instantiates);
 * replay with gridlp_graph_launch on any stream, free with
 * gridlp_graph_destroy. Kernel arguments are captured by value; the step
 * parameters are read from d_step at replay, so one graph serves every
 * chunk of a solve (pdhg_engine.py:394-400). */
int gridlp_iterate_graph_create(const gridlp_src_t* primal_src, const gridlp_primal_t* pv,
                                const gridlp_src_t* dual_src, const gridlp_dual_t* dv,
                                gridlp_step_t* d_step, int32_t n_iters, uint32_t flags, void** graph_exec);
int gridlp_graph_launch(void* graph_exec, void* stream);
int gridlp_graph_destroy(void* graph_exec);

/* --- device-side main loop (iterate_epoch, pdhg_engine.py:364-476) ----------
 * A CUDA graph with a WHILE conditional node whose body is one KKT interval
 * — the chunk of iterations, the KKT / restart-probe pass and
 * gridlp_loop_graph_decide's one-thread kernel — so consecutive intervals run
 * back to back without a host round trip. The decide kernel evaluates the
 * reference's per-pass logic on the pass's reduction slots exactly as the
 * host does (solver_driver / pdhg_engine expressions, IEEE-rounded sqrt and
 * divisions): relative KKT report, numerical failure, termination at the
 * tolerance, the fixed-point error and restart_decision (pdhg_engine.py:
 * 245-282), the iteration limit; the body repeats while none of them stops it
 * and fewer than max_passes passes ran. Each pass's slot values go to a ring
 * (GRIDLP_LOOP_REC doubles per pass) from which the host replays its
 * bookkeeping (reports, log lines, ledger, restart handling) after the
 * launch. Single-block grids only.
 *
 * Build: gridlp_loop_graph_begin starts capturing `stream` into the body;
 * the caller then issues the interval's launches on `stream`;
 * gridlp_loop_graph_decide appends the decide kernel; gridlp_loop_graph_end
 * instantiates (launch with gridlp_graph_launch, free with
 * gridlp_graph_destroy). gridlp_loop_graph_abort ends a failed capture. */
#define GRIDLP_LOOP_REC 12   /* kkt_rows[4], kkt_cols[4], probe[2], fp, stop flag */
typedef struct gridlp_loop {
  /* host-written before each launch */
  double eta, omega;                     /* constant between restarts */
  double bnorm, cnorm, obj_const, tolerance;
  double beta_sufficient, beta_necessary, beta_artificial;
  double base_fp, prev_fp;               /* valid when has_base / has_prev */
  int64_t total, inner_k;                /* iterations / Halpern counter before the launch */
  int64_t max_iterations, kkt_interval;
  int64_t max_passes;                    /* ring capacity: stop after this many passes */
  int32_t has_base, has_prev;
  int32_t restarts;                      /* EngineConfig.restarts */
  int32_t slot_rows, slot_cols, slot_probe;   /* reduction slots (rows of GRIDLP_MAX_RED doubles) */
  /* device-written */
  int64_t passes;                        /* passes completed by the launch (host sets 0) */
  int32_t stopped;
  int32_t reserved;
} gridlp_loop_t;
int gridlp_loop_graph_begin(void* stream, void** ctx);
int gridlp_loop_graph_decide(void* ctx, const double* slots, gridlp_loop_t* d_loop, double* d_ring);
int gridlp_loop_graph_end(void* ctx, void** graph_exec);
int gridlp_loop_graph_abort(void* ctx);
size_t gridlp_persistent_scratch_bytes(void);
/* n_iters fused iterations of a TINY single-block LP in ONE thread-block
 * cluster launch (8 CTAs x 512 threads): x_bar / y replicated in every CTA's shared
 * memory, each CTA's slices of A and A^T with their row operands resident
 * there, owners broadcast their new entries through distributed shared
 * memory, hardware cluster barriers between the products. Bit-identical to
 * gridlp_pdhg_iterate. `plan` (host memory, GRIDLP_CLUSTER_PLAN_LEN int64)
 * comes from gridlp_cluster_plan for the same matrices: entry-balanced slice
 * ranges per CTA and the shared memory per CTA; it reads the slice offsets
 * (synchronous D2H, once per matrix pair — outside any graph capture) and
 * returns GRIDLP_ERR_UNSUPPORTED when the LP does not fit one cluster's
 * shared memory or has long rows / column bands (use gridlp_pdhg_iterate). */
#define GRIDLP_CLUSTER_PLAN_LEN 35
/* The KKT / restart-probe pass fused into a cluster launch (evaluate_kkt
 * and the restart probe, pdhg_engine.py:310-346, :419-427): after the
 * iterations the same shared-memory slices give A x (KKT rows), A^T y (KKT
 * columns, x_probe_bar) and, with mode 2, A x_probe_bar (probe). Each row's
 * reduction terms land in t_rows [4 m] / t_cols [4 n] / t_probe [2 m] in
 * the gridlp_red_t.terms layout (term q of row r at q * rows + r); reduce
 * each with gridlp_reduce_terms — the same sums as the unfused ops. ax [m]
 * and xpb [n] receive A x and x_probe_bar as gridlp_op_kkt_rows /
 * gridlp_op_kkt_cols would write them. */
typedef struct gridlp_cluster_kkt {
  int32_t mode;            /* 0: no pass, 1: KKT rows + cols, 2: + restart probe */
  int32_t reserved;
  double* t_rows;
  double* t_cols;
  double* t_probe;
  double* ax;
  double* xpb;
} gridlp_cluster_kkt_t;
int gridlp_cluster_plan(const gridlp_src_t* primal_src, const gridlp_src_t* dual_src, int64_t* plan,
                        int64_t plan_len);
int gridlp_pdhg_iterate_cluster(const gridlp_src_t* primal_src, const gridlp_primal_t* pv,
                                const gridlp_src_t* dual_src, const gridlp_dual_t* dv,
                                gridlp_step_t* d_step, int32_t n_iters, uint32_t flags,
                                const int64_t* plan, const gridlp_cluster_kkt_t* kkt_pass, void* stream);
/* Fixed-order reduction of per-row terms (nred = 1, 2 or 4 per row, term q
 * of row r at terms[q * n + r]) into red->out[0..nred): the canonical
 * reduction every fused op uses (terms_reduce + final reduce). */
int gridlp_reduce_terms(const double* terms, int64_t n, int32_t nred, const gridlp_red_t* red, void* stream);
int gridlp_pdhg_iterate_persistent(const gridlp_src_t* primal_src, const gridlp_primal_t* pv,
                                   const gridlp_src_t* dual_src, const gridlp_dual_t* dv,
                                   gridlp_step_t* d_step, int32_t n_iters, uint32_t flags,
                                   void* scratch, void* stream);

/* --- one-off device preprocessing (csrc/gridlp_setup.cu) -----------------
 * Replaces permute_problem / distribute / slice_block / transpose
 * (partition.py:262-319, sparse_kernels.py:27-58; the from_coo lexsort of
 * lp_model.py:121-141 is the reference's setup hot spot). All outputs are
 * deterministic. `ws` is caller-allocated scratch of at least
 * gridlp_setup_workspace_bytes(items, segments) bytes. */
size_t gridlp_setup_workspace_bytes(int64_t max_items, int64_t max_segments);

/* Row counts of one grid block: band row lr is source row band_rows[lr]; an
 * entry belongs to the block when inv_col[col] is in [c0, c1). Writes the
 * block's row pointers (exclusive scan, out_ptr[nrows] = block nnz). */
int gridlp_block_count(const int64_t* src_ptr, const int32_t* src_col, const int64_t* band_rows,
                       int64_t nrows, const int32_t* inv_col, int32_t c0, int32_t c1,
                       int32_t* out_ptr, void* ws, size_t ws_bytes, void* stream);

/* Entries of the block with local columns inv_col[col] - c0, each row sorted
 * by column (== the reference's from_coo order after permutation). */
int gridlp_block_fill(const int64_t* src_ptr, const int32_t* src_col, const double* src_val,
                      const int64_t* band_rows, int64_t nrows, const int32_t* inv_col, int32_t c0,
                      int32_t c1, const int32_t* out_ptr, int64_t nnz, int32_t* out_col,
                      double* out_val, void* ws, size_t ws_bytes, void* stream);

/* Explicit CSR transpose with sorted columns (sparse_kernels.py:27-36). */
int gridlp_csr_transpose(const int32_t* ptr, const int32_t* col, const double* val, int64_t nrows,
                         int64_t ncols, int64_t nnz, int32_t* t_ptr, int32_t* t_col, double* t_val,
                         void* ws, size_t ws_bytes, void* stream);

/* counts[c] = entries with column c (exact histogram; the column lengths
 * that order the engine's internal column order). */
int gridlp_col_counts(const int32_t* col, int64_t nnz, int64_t ncols, int32_t* counts, void* stream);

/* out row r = row row_order[r] of the input (identity when NULL) with every
 * column index c replaced by col_label[c] (identity when NULL); entries keep
 * their order, so row sums are unchanged. Used to put a block in the
 * engine's internal length-sorted row/column order. */
int gridlp_csr_permute(const int32_t* ptr, const int32_t* col, const double* val, int64_t nrows,
                       const int32_t* row_order, const int32_t* col_label, int32_t* out_ptr,
                       int32_t* out_col, double* out_val, void* ws, size_t ws_bytes, void* stream);

/* SELL-32 plan for the rows of length <= light_row_max: lane_info
 * [32*ceil(nrows/32)], slice_off [ceil(nrows/32)+1], rank_of [nrows]; the
 * longer rows go to long_rows [nrows] / long_ptr [nrows+1]; sizes (device
 * int64[3]) = {SELL elements, long rows, long-row nonzeros}. */
int gridlp_sell_plan(const int32_t* ptr, int64_t nrows, int32_t light_row_max, int32_t* lane_info,
                     int64_t* slice_off, int32_t* rank_of, int32_t* long_rows, int32_t* long_ptr,
                     int64_t* sizes, void* ws, size_t ws_bytes, void* stream);

/* SELL-32 fill from a CSR and its plan (padding zeroed). */
int gridlp_sell_fill(const int32_t* ptr, const int32_t* col, const double* val, int64_t nrows,
                     int32_t light_row_max, const int64_t* slice_off, const int32_t* rank_of,
                     const int32_t* long_rows, const int32_t* long_ptr, int64_t num_long,
                     int32_t* sell_col, double* sell_val, int64_t sell_elems, int32_t* long_col,
                     double* long_val, void* stream);

/* --- device generators (csrc/gridlp_gen.cu) --------------------------------
 * Synthetic LPs of the BASELINE configs with no counterpart in the
 * reference's generators.py (cfg3 power-law, cfg4 multi-commodity flow).
 * Every random number is u(seed, stream, a, b) = (mix(mix(mix(seed *
 * 0x100000001B3 + stream) ^ a) ^ b) >> 11) * 2^-53 with mix = splitmix64's
 * finaliser, so instances are independent of grid, launch shape and device
 * and oracle/synth_oracle.py reproduces them bit for bit. */
size_t gridlp_gen_workspace_bytes(int64_t max_items, int64_t max_rows);
/* out = exclusive prefix sum of in[0..n) (n < 2^31). */
int gridlp_gen_scan64(const int64_t* in, int64_t* out, int64_t n, void* ws, size_t ws_bytes, void* stream);
/* Power-law column samples: entry k of row r (alloc_ptr[r] + k) gets
 * c = clamp(floor((1 + u(seed,1,r,k) kappa)^5) - 1, 0, n-1). */
int gridlp_gen_powerlaw_sample(uint64_t seed, const int64_t* alloc_ptr, int64_t m, int64_t n, double kappa,
                               int32_t* cols, void* stream);
/* Uniform column samples: entry k of row r gets floor(u(seed,1,r,k) n). */
int gridlp_gen_uniform_sample(uint64_t seed, const int64_t* alloc_ptr, int64_t m, int64_t n, int32_t* cols,
                              void* stream);
/* Planted optimum (cfg5): primal point x* and reduced cost r* of columns
 * j0 .. j0+n-1 (30 % at the lower bound with r* > 0, 10 % at the upper
 * bound with r* < 0, the rest interior with r* = 0). */
int gridlp_gen_planted_cols(uint64_t seed, int64_t j0, int64_t n, double lo, double hi, double* x, double* r,
                            void* stream);
/* Planted duals y* and row bounds around b = A x* for rows i0 .. i0+m-1
 * (35 % lower-active with y* > 0, 35 % upper-active with y* < 0, 30 %
 * inactive with y* = 0). */
int gridlp_gen_planted_rows(uint64_t seed, int64_t i0, int64_t m, const double* b, double* y, double* lo,
                            double* hi, void* stream);
/* Sharded cfg5 generation (no device ever holds the whole matrix):
 * d draws per row for rows r0 .. r0+m-1 (row-major, floor(u(seed,1,r,k) n)). */
int gridlp_gen_band_draws(uint64_t seed, int64_t r0, int64_t m, int32_t d, int64_t n, int32_t* cols,
                          void* stream);
/* b[q] = A x* of full (sorted, possibly repeated) row r0+q, sequential in
 * column order from +0.0 — the one-piece instance's value. */
int gridlp_gen_planted_row_dot(const int64_t* ptr, const int32_t* sorted, int64_t m, int64_t r0, uint64_t seed,
                               double lo, double hi, double* b, void* stream);
/* acc[c] += value * y*(row) over the transposed chunk block, rows ascending
 * (continues the sequential column sum Aᵀ y* across row chunks). */
int gridlp_gen_col_accumulate(const int32_t* tptr, const int32_t* trows, const double* tvals, int64_t ncols,
                              int64_t r0, uint64_t seed, double* acc, void* stream);
/* out = a + b (c = Aᵀ y* + r*). */
int gridlp_gen_add(const double* a, const double* b, int64_t n, double* out, void* stream);
/* Sort the keys of every row segment ptr[r]..ptr[r+1] ascending. */
int gridlp_gen_sort_rows(const int64_t* ptr, int64_t m, int64_t items, const int32_t* keys_in,
                         int32_t* keys_out, void* ws, size_t ws_bytes, void* stream);
/* counts[r] = distinct keys of sorted row r inside [c0, c1); counts[m] = 0. */
int gridlp_gen_dedupe_count(const int64_t* ptr, const int32_t* sorted, int64_t m, int32_t c0, int32_t c1,
                            int64_t* counts, void* stream);
/* Compact those keys into out_ptr's rows as local columns c - c0; value of
 * global entry (r0 + r, c) is 2 u(seed,2,r0+r,c) - 1. */
int gridlp_gen_dedupe_fill(const int64_t* ptr, const int32_t* sorted, int64_t m, int64_t r0, int32_t c0,
                           int32_t c1, const int64_t* out_ptr, uint64_t seed, int32_t* out_cols,
                           double* out_vals, void* stream);
/* out_i = lo + (hi - lo) u(seed, stream_id, i0 + i, 0). */
int gridlp_gen_uniform(uint64_t seed, uint64_t stream_id, int64_t i0, int64_t n, double lo, double hi,
                       double* out, void* stream);
/* y = A x with each row summed left to right from +0.0 (scipy csr_matvec
 * order, the reference's rhs = A x_hat, generators.py:125). */
int gridlp_csr_spmv_seq(const int64_t* ptr, const int32_t* cols, const double* vals, int64_t m,
                        const double* x, double* y, void* stream);
/* Feasible row bounds around b: with probability ineq a row is ranged,
 * [b - U[0.1,1), b + U[0.1,1)), else lo = hi = b (generators.py:120-142). */
int gridlp_gen_row_bounds(uint64_t seed, int64_t m, double ineq, const double* b, double* lo, double* hi,
                          void* stream);
/* Multi-commodity flow matrix: lens[r] of the K*V conservation rows and E
 * coupling rows (lens[m] = 0, scan for row_ptr), then the fill. */
int gridlp_gen_mcf_row_lengths(int64_t K, int64_t V, int64_t E, const int32_t* adj_ptr, int64_t* lens,
                               void* stream);
int gridlp_gen_mcf_fill(int64_t K, int64_t V, int64_t E, const int32_t* adj_ptr, const int32_t* adj_arc,
                        const int8_t* adj_sign, const int64_t* row_ptr, int32_t* cols, double* vals,
                        void* stream);

/* --- diagonal preconditioning (csrc/gridlp_scale.cu) -------------------------
 * Ruiz equilibration + Pock-Chambolle scaling of A, opt-in
 * (SolverConfig.scaling; the reference has none). Matrices here
 * are the original problem's CSR (int64 row pointers, int32 columns). */
/* out[r] = max |a_rk| over row r. */
int gridlp_row_absmax(const int64_t* ptr, const double* val, int64_t m, double* out, void* stream);
/* out[r] = sum |a_rk|^power over row r (power 1 or 2), sequential in entry order. */
int gridlp_row_abssum(const int64_t* ptr, const double* val, int64_t m, int32_t power, double* out,
                      void* stream);
/* out[c] = max |a_kc| over column c (order-free atomic max). */
int gridlp_col_absmax(const int32_t* col, const double* val, int64_t nnz, int64_t ncols, double* out,
                      void* stream);
/* step[i] = 1/sqrt(s[i]) (1 when s[i] = 0); d[i] *= step[i]. */
int gridlp_update_scale(const double* s, int64_t n, double* d, double* step, void* stream);
/* a_rc <- (dr[r] a_rc) dc[c] in place. */
int gridlp_scale_matrix(const int64_t* ptr, const int32_t* col, double* val, int64_t m, const double* dr,
                        const double* dc, void* stream);
/* v[i] <- v[i] * d[i] (divide = 0) or v[i] / d[i] (divide = 1). */
int gridlp_scale_vector(double* v, const double* d, int64_t n, int32_t divide, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* GRIDLP_B200_H */
