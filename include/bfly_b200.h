/*
 * bfly_b200.h -- C ABI of the B200-native butterfly construction library.
 *
 * Drop-in boundary for the reference's construction path
 * (/root/reference/proj/include/bfly/).  Every entry point names the reference
 * interface it replaces.  Plain pointers and sizes only; no exceptions cross
 * this boundary -- every call returns a bfly_status and bfly_last_error()
 * holds the message (the reference's exception hierarchy,
 * core.hpp:43-60, maps 1:1 onto the status codes).
 *
 * Complex data is interleaved (re, im) column-major, like Eigen's
 * Matrix<std::complex<double>> storage the reference uses.
 */
#ifndef BFLY_B200_H
#define BFLY_B200_H

#include <stdint.h>

#if defined(__GNUC__)
#define BFLY_API __attribute__((visibility("default")))
#else
#define BFLY_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

/* status codes: core.hpp:43-60 (precondition, dimension, sequencing, format,
 * conditioning) + device/collective failures */
typedef enum {
  BFLY_OK = 0,
  BFLY_PRECONDITION = 1,
  BFLY_DIMENSION = 2,
  BFLY_SEQUENCING = 3,
  BFLY_FORMAT = 4,
  BFLY_CONDITIONING = 5,
  BFLY_CUDA = 6,
  BFLY_NCCL = 7,
} bfly_status;

/* scalar types: scalar_traits (core.hpp:29-39) covers real64/complex128;
 * complex64 is the B200-only single-precision variant (BASELINE config 4). */
typedef enum { BFLY_Z = 0, BFLY_C = 1, BFLY_D = 2 } bfly_scalar;

/* transpose selector: apply (operators.hpp:27-31) / apply_transpose (:34-38) /
 * apply_adjoint (:59-66) */
typedef enum { BFLY_N = 0, BFLY_T = 1, BFLY_H = 2 } bfly_trans;

typedef struct bfly_ctx bfly_ctx;
typedef struct bfly_tree bfly_tree;
typedef struct bfly_op bfly_op;
typedef struct bfly_bf bfly_bf;
typedef struct bfly_factorizer bfly_factorizer;

BFLY_API const char* bfly_last_error(void);
BFLY_API const char* bfly_version(void);

/* ---------------------------------------------------------------- context */
/* One context per GPU/process: streams, memory pool, counters.
 * (reference: none -- it is single-process CPU code) */
BFLY_API int bfly_ctx_create(int device, bfly_ctx** out);
BFLY_API int bfly_ctx_destroy(bfly_ctx* ctx);
/* kernels launched by the library on this context since creation */
BFLY_API int64_t bfly_ctx_launches(const bfly_ctx* ctx);
BFLY_API int bfly_ctx_synchronize(bfly_ctx* ctx);
/* raw stream handle (cudaStream_t) the library launches on */
BFLY_API void* bfly_ctx_stream(bfly_ctx* ctx);
/* per-kernel device timing with CUDA events on the library stream:
 * enable = 1 on, 0 off, -1 off and clear.  The report is a JSON object
 * {kernel: {launches, ms, flops, bytes}}; returns the length needed. */
BFLY_API int bfly_ctx_profile(bfly_ctx* ctx, int enable);
BFLY_API int64_t bfly_ctx_profile_report(bfly_ctx* ctx, char* buf, int64_t len);
/* Multi-GPU: join an NCCL communicator (ncclUniqueId bytes from rank 0).
 * Probes and butterfly blocks are sharded across ranks; each level's new
 * blocks are all-gathered. */
BFLY_API int bfly_comm_unique_id(uint8_t* id_out /* 128 bytes */);
BFLY_API int bfly_ctx_set_comm(bfly_ctx* ctx, int rank, int world, const uint8_t* nccl_id);
/* Host-staged transport: the same sharded schedule with every exchange staged
 * through pinned host memory and handed to the caller's collectives (e.g.
 * torch.distributed over gloo).  For ranks that share one GPU (NCCL rejects
 * two ranks on one device) or lack peer access; the library synchronizes its
 * stream before each exchange, so no kernel ever waits on another rank.
 * Every function is collective (all ranks call it in the same order) and
 * returns 0 on success.  Host buffers are library-owned, valid for the call.
 *   allgather: recv (world * bytes) = concat over ranks of send (bytes)
 *   allreduce: in place on count elements; dtype 0 int32, 1 float64,
 *              2 float32; op 0 sum, 1 max
 *   sendrecv:  one group of point-to-point transfers (ncclGroupStart ..
 *              ncclGroupEnd semantics: all posted, then all completed) */
typedef struct bfly_host_comm {
  void* user;
  int (*allgather)(void* user, const void* send, void* recv, int64_t bytes);
  int (*allreduce)(void* user, void* buf, int64_t count, int dtype, int op);
  int (*sendrecv)(void* user, int nsend, const int32_t* send_peer, void* const* send_buf, const int64_t* send_bytes,
                  int nrecv, const int32_t* recv_peer, void* const* recv_buf, const int64_t* recv_bytes);
} bfly_host_comm;
BFLY_API int bfly_ctx_set_host_comm(bfly_ctx* ctx, int rank, int world, const bfly_host_comm* hc);
/* rank / world of the context's transport (0 / 1 when none); transport 0 none,
 * 1 NCCL, 2 host-staged */
BFLY_API int bfly_ctx_comm_info(const bfly_ctx* ctx, int* rank, int* world, int* transport);

/* ------------------------------------------------------------------- trees */
/* PartitionTree::build (tree.hpp:75-101); coords n x 3 row-major */
BFLY_API int bfly_tree_build(int dim, int64_t n, const double* coords, int levels, bfly_tree** out);
/* PartitionTree::set_permutation (tree.hpp:153-159) with the serialized table
 * layout (serialize.hpp:64-71): perm[n], ranges = concat_l (2^l + 1 entries) */
BFLY_API int bfly_tree_from_table(int64_t n, int levels, const int64_t* perm, const int64_t* ranges, bfly_tree** out);
BFLY_API int bfly_tree_info(const bfly_tree* t, int64_t* n, int* levels);
BFLY_API int bfly_tree_table(const bfly_tree* t, int64_t* perm, int64_t* ranges);
BFLY_API void bfly_tree_destroy(bfly_tree* t);
/* PartitionTree::depth_for (tree.hpp:163-168) */
BFLY_API int bfly_depth_for(int64_t n, int64_t leaf_cap);

/* ------------------------------------------------------- point generators */
/* Seeded point sets of the BASELINE configs (host). */
BFLY_API void bfly_points_uniform(int64_t n, uint64_t seed, uint64_t tag, double lo, double hi, double* out);
BFLY_API void bfly_points_plate(int64_t side, double z, double* out);
BFLY_API void bfly_points_half_circle(int64_t n, int upper, double* out);

/* --------------------------------------------------------------- operators */
/* BlackBoxOperator<Scalar> (operators.hpp:17-56).  Built-in kinds evaluate
 * the kernel on the fly on the GPU (the pattern of operators.hpp:430-439). */
typedef enum {
  BFLY_OP_DENSE = 0,     /* DenseOperator (operators.hpp:68-85) */
  BFLY_OP_NUFFT = 1,     /* exp(2 pi i x_i xi_j)                 (config 0) */
  BFLY_OP_PLATES = 2,    /* exp(i k r) / (4 pi r), 3D            (config 1) */
  BFLY_OP_CIRCLE = 3,    /* exp(i k r) / r, 2D                   (config 2) */
  BFLY_OP_COMPOSE = 4,   /* F2 * F1, sequential products         (config 3) */
  BFLY_OP_BUTTERFLY = 5, /* ButterflyOperator (operators.hpp:105-122) (config 4) */
  BFLY_OP_CALLBACK = 6,  /* user black box (stream-ordered callback) */
} bfly_op_kind;

/* User black box.  Y (rows_out x k, ldy) = op(A) X (rows_in x k, ldx); trans is
 * BFLY_N or BFLY_T (plain transpose -- the library derives the adjoint by
 * conjugation exactly as apply_adjoint, operators.hpp:59-66).  Buffers are
 * device pointers owned by the library, valid for the duration of the call;
 * the callback must be ordered on `stream` (a cudaStream_t). */
typedef int (*bfly_apply_fn)(void* user, int trans, const void* x_dev, int64_t ldx, void* y_dev,
                             int64_t ldy, int64_t k, void* stream);

/* Structured-probe-aware user black box.  Same contract as
 * bfly_apply_fn plus the probe's nonzero input rows: x_dev is full height in
 * operator (original) row order and zero outside [nz_row_begin, nz_row_end),
 * so a reference-style body may ignore the range, while a range-aware body
 * reads only those rows and skips the zero work (the reference pads the probe
 * and multiplies the zeros, reconstruct.hpp:72-85, operators.hpp:17-56).  The
 * library calls it once per structured probe (a contiguous range exists when
 * the probe side's tree is the identity, i.e. points in tree order; otherwise
 * the range is [0, rows_in)), and with [0, rows_in) for dense inputs. */
typedef int (*bfly_apply_range_fn)(void* user, int trans, const void* x_dev, int64_t ldx, void* y_dev,
                                   int64_t ldy, int64_t k, int64_t nz_row_begin, int64_t nz_row_end, void* stream);

/* tgt (m x 3) and src (n x 3) row-major host points, already in tree order */
BFLY_API int bfly_op_kernel(bfly_ctx* ctx, int kind, int64_t m, int64_t n, const double* tgt, const double* src,
                   double wavenumber, int scalar, bfly_op** out);
/* A = f2 * f1; takes ownership of both factors */
BFLY_API int bfly_op_compose(bfly_ctx* ctx, bfly_op* f2, bfly_op* f1, bfly_op** out);
/* a: host m x n column-major interleaved complex (or real for BFLY_D) */
BFLY_API int bfly_op_dense(bfly_ctx* ctx, int64_t m, int64_t n, const double* a, int scalar, bfly_op** out);
/* wraps a butterfly as a black box; takes ownership */
BFLY_API int bfly_op_butterfly(bfly_ctx* ctx, bfly_bf* bf, bfly_op** out);
BFLY_API int bfly_op_callback(bfly_ctx* ctx, int64_t m, int64_t n, int scalar, bfly_apply_fn fn, void* user,
                     bfly_op** out);
BFLY_API int bfly_op_callback_ranged(bfly_ctx* ctx, int64_t m, int64_t n, int scalar, bfly_apply_range_fn fn,
                                     void* user, bfly_op** out);
BFLY_API int bfly_op_info(const bfly_op* op, int64_t* m, int64_t* n, int* scalar, int* kind);
/* apply / apply_transpose / apply_adjoint.  on_device = 0: host buffers (copied
 * in and out inside the call); 1: device pointers, stream-ordered. */
BFLY_API int bfly_op_apply(bfly_op* op, int trans, const void* x, int64_t ldx, void* y, int64_t ldy, int64_t k,
                  int on_device);
/* forward_columns / transpose_columns (operators.hpp:41-47) */
BFLY_API int bfly_op_counters(const bfly_op* op, int64_t* fwd, int64_t* tr);
BFLY_API int bfly_op_reset_counters(bfly_op* op);
BFLY_API void bfly_op_destroy(bfly_op* op);

/* ---------------------------------------------------------- reconstruction */
/* ReconstructionConfig (reconstruct.hpp:10-36) + batching knob */
typedef struct bfly_recon_cfg {
  double tolerance;
  int64_t oversampling;
  int64_t rank_guess;
  int32_t levels;
  int32_t center;       /* -1: floor(L/2) */
  uint64_t seed;
  int64_t hard_cap;     /* -1: min(m, n) */
  int32_t threads;      /* accepted for API parity; the GPU path ignores it */
  int32_t literal_transpose_core;
  int64_t max_batch_probes; /* probes per black-box launch; <= 0: a whole level */
  int32_t virtual_ranks;    /* >1: execute the rank-sharded schedule for this many ranks in one
                               process (tests the multi-GPU exchange on one GPU); 0/1: off */
  int32_t reserved_;
} bfly_recon_cfg;

BFLY_API void bfly_cfg_default(bfly_recon_cfg* cfg);

/* PhaseStat / FactorizationLog (reconstruct.hpp:87-120) */
#define BFLY_MAX_PHASES 64
typedef struct bfly_phase {
  char name[32];
  int64_t forward_columns;
  int64_t transpose_columns;
  double seconds;
  int32_t rounds;
  int64_t probe_width;
  /* CPQR rank margin at the truncation cut (diagnostic; SURVEY 7 hard part 1):
   * min over the phase's blocks (leaf phases: the kept round) of
   * min(|R_{k-1}| / thr - 1, 1 - |R_k| / thr), thr = 0.25 tol |R_00|
   * (linalg.hpp:74-77, reconstruct.hpp:342-348); +inf when no block was
   * truncated.  Near 0 = a rank that rounding could flip.  Multi-process:
   * over this process's blocks. */
  double rank_margin;
} bfly_phase;

typedef struct bfly_log {
  int32_t nphases;
  bfly_phase phases[BFLY_MAX_PHASES];
  uint64_t peak_probe_bytes;
  int64_t peak_concurrent_probes;
  int32_t rank_capped;
  double total_seconds;
  double flops;         /* algorithmic flops of the construction */
  double kernel_evals;  /* black-box kernel-entry evaluations */
  /* 1 when a kernel entry fell outside the int8-slice range and the whole
   * factorization was recomputed on the FP64 path (same results, ~2x time) */
  int32_t products_recomputed;
} bfly_log;

/* factorize() (reconstruct.hpp:412-419) */
BFLY_API int bfly_factorize(bfly_ctx* ctx, bfly_op* op, const bfly_tree* row_tree, const bfly_tree* col_tree,
                   const bfly_recon_cfg* cfg, bfly_bf** out, bfly_log* log);
/* Factorizer phase-stepping API (reconstruct.hpp:145-321) */
BFLY_API int bfly_factorizer_create(bfly_ctx* ctx, bfly_op* op, const bfly_tree* row_tree, const bfly_tree* col_tree,
                           const bfly_recon_cfg* cfg, bfly_factorizer** out);
BFLY_API int bfly_factorizer_leaf_row_bases(bfly_factorizer* f);
BFLY_API int bfly_factorizer_leaf_col_bases(bfly_factorizer* f);
BFLY_API int bfly_factorizer_transfer_level_w(bfly_factorizer* f, int l);
BFLY_API int bfly_factorizer_transfer_level_r(bfly_factorizer* f, int l);
BFLY_API int bfly_factorizer_complete(const bfly_factorizer* f);
/* hands the finished butterfly to the caller (validates it first) */
BFLY_API int bfly_factorizer_take(bfly_factorizer* f, bfly_bf** out, bfly_log* log);
BFLY_API void bfly_factorizer_destroy(bfly_factorizer* f);

/* estimate_error (reconstruct.hpp:423-434) */
BFLY_API int bfly_estimate_error(bfly_op* op, bfly_bf* bf, int64_t k, uint64_t seed, double* err);

/* Level-wise residual sums of bf against a dense copy of op (desk scale: the
 * operator is densified on the GPU), reconstruct.hpp:443-503 u_side_residual /
 * v_side_residual / center_residual:
 *   u_res[L - l]  for l = L .. l_m   sum_b ||K_b - U U^H K_b||_F^2
 *   v_res[l]      for l = 0 .. l_m   sum_b ||K_b - K_b V V^H||_F^2
 *   *center                          sum_b ||K_b - U (U^H K_b V) V^H||_F^2
 *   *knorm2                          ||K||_F^2
 * (the error-bound check of Theorems 5.1-5.3, tools/bfly_cli.cpp:208-235) */
BFLY_API int bfly_residuals(bfly_op* op, bfly_bf* bf, double* u_res, double* v_res, double* center, double* knorm2);

/* ---------------------------------------------------------------- butterfly */
/* HybridButterfly::apply / apply_transpose / apply_adjoint (butterfly.hpp:71-193) */
BFLY_API int bfly_apply(bfly_bf* bf, int trans, const void* x, int64_t ldx, void* y, int64_t ldy, int64_t k,
               int on_device);
/* Process layouts of the apply (inc/layout.hpp).  kind: 0 column, 1 row,
 * 2 hybrid; processes a power of two <= 2^L.
 * bfly_comm_cost: closed-form CommCostReport (comm_cost, layout.hpp:70-88)
 *   out[4] = exchange volume, exchange messages, all-to-all volume,
 *   all-to-all messages (scalars per input column and process).
 * bfly_layout_owners: assign_ownership (layout.hpp:139-188) without a
 *   butterfly; out[(L+3) 2^L] = u leaves, v leaves, R levels center..L-1,
 *   W levels 1..center, centre cores (flat block index tau*2^(L-l)+nu);
 *   returns the length (out == NULL: length only) or -status.
 * bfly_apply_layout: the apply (trans N or H) executed over the layout: with
 *   a communicator (bfly_ctx_set_comm) one process per GPU exchanging
 *   coefficient blocks by NCCL send/recv, else `processes` virtual processes
 *   in turn on this GPU; x full input, y full output on every process.
 *   report[6] = the four simulated_parallel_apply tallies
 *   (layout.hpp:190-261), then the measured scalars per column received by
 *   the busiest process and in total. */
BFLY_API int bfly_comm_cost(int kind, int levels, int64_t rank, int64_t processes, double* out);
BFLY_API int64_t bfly_layout_owners(int kind, int levels, int center, int64_t processes, int32_t* out);
BFLY_API int bfly_apply_layout(bfly_bf* bf, int trans, int kind, int64_t processes, const void* x, int64_t ldx, void* y,
                               int64_t ldy, int64_t k, int on_device, double* report);
BFLY_API int bfly_bf_info(const bfly_bf* bf, int* levels, int* center, int64_t* m, int64_t* n, int64_t* nnz,
                 int64_t* max_rank, int* scalar);
/* u ranks for levels center..L, then v ranks for levels 0..center (2^L each,
 * index tau*2^(L-l)+nu, butterfly.hpp:38-66) */
BFLY_API int64_t bfly_rank_profile(const bfly_bf* bf, int32_t* out);
/* .bfh container (serialize.hpp:103-191; proj/docs/formats.md:3-54) */
BFLY_API int64_t bfly_serialize(const bfly_bf* bf, uint8_t* buf);
BFLY_API int bfly_deserialize(bfly_ctx* ctx, const uint8_t* buf, int64_t nbytes, int scalar, bfly_bf** out);
/* seeded synthetic butterfly (synth_butterfly, operators.hpp:131-178,
 * generalised to leaf size b and rank r; perturb = relative Gaussian noise) */
BFLY_API int bfly_synth_butterfly(bfly_ctx* ctx, int levels, int64_t leaf, int64_t rank, uint64_t seed, int scalar,
                         double perturb, bfly_bf** out);
BFLY_API int bfly_bf_convert(bfly_bf* bf, int scalar, bfly_bf** out);
BFLY_API void bfly_bf_destroy(bfly_bf* bf);

/* ---------------------------------------------------------------- shard plan */
/* How the multi-GPU construction splits a level (host logic): contiguous chunk
 * of n units for a rank, and the block indices a rank produces (side 0 leaves,
 * 1 W level (row probes), 2 R level (column probes)); returns the count. */
BFLY_API int bfly_shard_chunk(int64_t n, int world, int rank, int64_t* begin, int64_t* end);
BFLY_API int64_t bfly_shard_blocks(int levels, int level, int side, int world, int rank, int64_t* out);
/* Diagnostics for a scaling projection: device milliseconds of every rank's
 * share of every phase of the last factorization run with virtual_ranks > 1
 * and BFLY_VRANK_TIMING=1 (row-major, virtual_ranks entries per phase, phases
 * in log order); returns the entry count, copies up to cap entries. */
BFLY_API int64_t bfly_vrank_times(double* out, int64_t cap);

/* ------------------------------------------------------------- dense helpers */
/* gaussian_matrix (linalg.hpp:16-25) generated on the device, copied to host */
BFLY_API int bfly_gaussian(bfly_ctx* ctx, int64_t rows, int64_t cols, uint64_t seed, int scalar, void* out_host);
BFLY_API uint64_t bfly_seed_mix(uint64_t seed, int nwords, const uint64_t* words);
/* pivoted_qr_truncate (linalg.hpp:62-80) on the device, batch of one */
BFLY_API int bfly_cpqr_truncate(bfly_ctx* ctx, int64_t rows, int64_t cols, const double* z_host, double eps,
                       double* q_host, int64_t* k_out);
/* pinv_solve (linalg.hpp:128-139) on the device, batch of one */
BFLY_API int bfly_pinv(bfly_ctx* ctx, int64_t rows, int64_t cols, const double* m_host, double tol, double* out_host);

#ifdef __cplusplus
}
#endif
#endif
