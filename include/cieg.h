/* cieg.h -- C ABI of the B200-native LOBPCG hot path.
 *
 * This is the drop-in boundary for the reference's C++ solver/operator API in
 * /root/reference/proj/include/ci/. Every entry point below names the
 * reference interface it replaces (file:line). Plain pointers and sizes only:
 * no C++ or torch types cross this boundary and no exception escapes it.
 * Every function returns a cieg_status; on failure cieg_last_error() holds
 * "<Type>: message" using the reference's ci::Error taxonomy
 * (proj/include/ci/errors.hpp:9-32), so a C++ layer can rethrow the matching
 * ci:: exception.
 *
 * Conventions
 *   - Block vectors are row-major n x k doubles (BlockVectors,
 *     proj/include/ci/block_vectors.hpp:19-54): the k components of one basis
 *     state are adjacent.
 *   - Small dense matrices (Grams, coefficient panels) are column-major
 *     doubles with leading dimension = rows (Eigen::MatrixXd default).
 *   - "_dev" pointers are device addresses on the context's GPU; "_host"
 *     pointers are host memory (pageable or pinned).
 *   - A context owns one CUDA stream; it is not re-entrant (one host thread
 *     at a time), mirroring the reference's single-threaded caller
 *     (SURVEY.md 8(b) Threading).
 */
#ifndef CIEG_H
#define CIEG_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  CIEG_OK = 0,
  CIEG_ERR_DIMENSION = 1,   /* ci::DimensionMismatch */
  CIEG_ERR_CONFIG = 2,      /* ci::ConfigError */
  CIEG_ERR_SUBSPACE = 3,    /* ci::SubspaceCollapse */
  CIEG_ERR_FORMAT = 4,      /* ci::FormatError */
  CIEG_ERR_INDEFINITE = 5,  /* ci::IndefiniteGram */
  CIEG_ERR_CUDA = 6,        /* device/runtime failure (no reference analogue) */
  CIEG_ERR_ARGUMENT = 7,    /* null handle / bad argument (ci::Error) */
  CIEG_ERR_BETA = 8         /* ci::BetaTooLarge */
} cieg_status;

/* Last error message of the calling thread ("" when none). */
const char* cieg_last_error(void);
/* Library version string. */
const char* cieg_version(void);

typedef struct cieg_ctx cieg_ctx;
typedef struct cieg_mat cieg_mat;
typedef struct cieg_prec cieg_prec;
typedef struct cieg_report cieg_report;
typedef struct cieg_host_csb cieg_host_csb;

/* ---- context --------------------------------------------------------- */
/* Bind a context (one CUDA stream) to a device. No reference analogue: the
 * reference is host-only. */
/* Device buffers on the context's GPU for integrators that hold host data
 * (the reference-side drop-in stages ci::BlockVectors through these).
 * cieg_memcpy kind: 0 host->device, 1 device->host, 2 device->device;
 * ordered on the context stream and synchronous. */
int cieg_device_alloc(cieg_ctx* ctx, uint64_t bytes, void** out);
int cieg_device_free(cieg_ctx* ctx, void* p);
int cieg_memcpy(cieg_ctx* ctx, void* dst, const void* src, uint64_t bytes, int kind);
int cieg_ctx_create(int device, cieg_ctx** out);
int cieg_ctx_destroy(cieg_ctx* ctx);
int cieg_ctx_synchronize(cieg_ctx* ctx);
/* cudaStream_t of the context, as void* (for callers that enqueue their own
 * work, e.g. torch.cuda.ExternalStream). */
void* cieg_ctx_stream(cieg_ctx* ctx);
/* 1: the preconditioner's FOM reproduces the reference's operation order
 * bit for bit (sequential dots, un-fused products); 0 (default): DMMA block
 * products and parallel fixed-order reductions (deterministic, ~1e-16
 * relative difference). Direct LU solves are reference-order in both. */
int cieg_ctx_set_exact_order(cieg_ctx* ctx, int exact);
/* SpMM (K1) mode: CIEG_SPMM_AUTO (default) = single pass for block widths
 * <= 8 on unsharded matrices, owner-computes otherwise; CIEG_SPMM_OWNER =
 * every stored tile streamed once per owner panel; CIEG_SPMM_SINGLE_PASS =
 * one pass per stored tile, H·X and Hᵀ·X from the same shared tile, the
 * transposed half reduced through per-tile partials (unsharded matrices;
 * shards stay owner-computes). All modes are deterministic. Replaces no
 * reference call: spmm (csb.cpp:118-193) has one code path. */
/* CIEG_SPMM_SLICED = the single pass on the int8 tensor cores (tcgen05):
 * H and X split into exact 8-bit integer slices (Ozaki scheme), int32
 * accumulators in TMEM, recombined in fp64 -- fp32 H with 128-row panels on
 * unsharded matrices; agrees with the fp64 modes to rounding (~1e-16), not
 * bit for bit. AUTO picks it for widths >= 9 where supported. */
enum { CIEG_SPMM_AUTO = 0, CIEG_SPMM_OWNER = 1, CIEG_SPMM_SINGLE_PASS = 2, CIEG_SPMM_SLICED = 3 };
int cieg_ctx_set_spmm_mode(cieg_ctx* ctx, int mode);
/* The K1 kernel the current mode runs for a 16-column chunk of width m on
 * this matrix: CIEG_SPMM_OWNER, CIEG_SPMM_SINGLE_PASS or CIEG_SPMM_SLICED
 * (instrumentation; builds the sliced kernel's slice planes on first use, so
 * calling it once after an upload moves that one-time setup out of the first
 * SpMM / solve). */
int cieg_spmm_effective_mode(cieg_ctx* ctx, cieg_mat* mat, uint32_t m, int* mode);
/* Number of kernels this context has launched (instrumentation). */
uint64_t cieg_ctx_launch_count(const cieg_ctx* ctx);

/* ---- matrix ------------------------------------------------------------ */
/* Flattened ci::CsbMatrix (proj/include/ci/csb.hpp:33-60): the lower-triangle
 * CSB block grid, block (I,J<=I) at linear index I(I+1)/2+J, entries of one
 * block contiguous and sorted by (row, col) with 16-bit block-local offsets.
 * entry_offsets has nb(nb+1)/2 + 1 prefix sums into rows/cols/values. */
typedef struct {
  uint32_t dim;
  uint32_t nb;                     /* CSB block count */
  int precision;                   /* 0 = single (values32), 1 = double (values64) */
  const uint32_t* block_boundaries;/* nb + 1 */
  const uint64_t* entry_offsets;   /* nb(nb+1)/2 + 1 */
  const uint16_t* rows;
  const uint16_t* cols;
  const void* values;              /* float or double per precision */
} cieg_csb_view;

/* Upload H once and re-tile it into the device format (row panels <= tile
 * edge, dense-able 32-bit packed tile-local indices, 64-bit offsets).
 * panel_bounds (npanels+1 entries, 0 .. dim) fixes the device panel grid; pass
 * NULL to derive it from group_bounds (ngroups+1 entries, e.g. a
 * GroupPartition's ranges) or, when both are NULL, from a fixed grid.
 * tile_edge is 64 or 128 (0 = choose). Replaces the host-side ownership of
 * CsbMatrix for spmm (proj/src/csb.cpp:182-193). */
int cieg_matrix_upload(cieg_ctx* ctx, const cieg_csb_view* csb,
                       const uint32_t* group_bounds, uint32_t ngroups,
                       uint32_t tile_edge, cieg_mat** out);
/* cieg_matrix_upload with extra mandatory device-panel boundaries cuts[ncuts]
 * (e.g. the truncation dimensions of cieg_multilevel_guess, so their leading
 * blocks can be viewed without copying). */
int cieg_matrix_upload_cuts(cieg_ctx* ctx, const cieg_csb_view* csb, const uint32_t* group_bounds,
                            uint32_t ngroups, uint32_t tile_edge, const uint32_t* cuts, uint32_t ncuts,
                            cieg_mat** out);
int cieg_matrix_destroy(cieg_mat* mat);
/* dim, stored nnz (lower incl. diagonal), device panels, device tiles,
 * tile edge, precision, device bytes of the tile stream. */
int cieg_matrix_info(const cieg_mat* mat, uint32_t* dim, uint64_t* nnz, uint32_t* npanels,
                     uint64_t* ntiles, uint32_t* tile_edge, int* precision, uint64_t* bytes);

/* U = (L + L^T - diag L) X  --  ci::spmm (proj/include/ci/csb.hpp:83,
 * proj/src/csb.cpp:182-193). x_dev, y_dev: row-major dim x m device arrays
 * (leading dimension m). Deterministic: every output row is reduced by one
 * owner in a fixed order (bitwise identical run to run). */
int cieg_spmm(cieg_ctx* ctx, const cieg_mat* mat, const double* x_dev, double* y_dev, uint32_t m);
/* Same with host buffers (pageable or pinned), synchronous on return. This is
 * the call a ci::spmm drop-in makes. Where the sliced kernel applies (an
 * unsharded fp32 H, m <= 16) the upload of X, the kernels and the download of
 * U are pipelined over chunks of row panels on the context's copy streams,
 * with results bitwise those of cieg_spmm; otherwise H2D, SpMM, D2H on the
 * context stream. */
int cieg_spmm_host(cieg_ctx* ctx, const cieg_mat* mat, const double* x_host, double* y_host,
                   uint32_t m);
/* `count` independent products U_i = H X_i through host buffers (pinned for
 * full overlap), pipelined over three device buffer sets: the upload of
 * X_{i+1} and the download of U_{i-1} run on the copy engines while K1
 * computes U_i. Same results as `count` calls of cieg_spmm_host. */
int cieg_spmm_host_batch(cieg_ctx* ctx, const cieg_mat* mat, const double* const* x_hosts, double* const* y_hosts,
                         uint32_t m, uint32_t count);

/* ---- row-block sharding over several GPUs ------------ */
/* Partition the rows over nranks at group boundaries (a group never straddles
 * two ranks, so each rank's tile diagonal is local), balanced by the stored
 * entries each owner streams (owner-computes: a rank reads its rows' tiles and
 * the tiles (I > P, P) whose transposed part lands in its rows).
 * row_bounds: nranks + 1 entries. halo_lo/halo_hi: the X rows rank r's SpMM
 * reads. Host-only (no device needed). The planner of the reference only
 * models this (planner.cpp:88-139). */
int cieg_shard_plan(const cieg_csb_view* csb, const uint32_t* group_bounds, uint32_t ngroups,
                    uint32_t tile_edge, uint32_t nranks, uint32_t* row_bounds, uint32_t* halo_lo,
                    uint32_t* halo_hi);
/* Upload the part of H that owner rows [row_lo, row_hi) need. cieg_spmm on
 * the result reads a full-length X (only rows [halo_lo, halo_hi) are touched)
 * and writes rows [row_lo, row_hi) of U into a LOCAL buffer (row_lo -> row 0). */
int cieg_matrix_upload_shard(cieg_ctx* ctx, const cieg_csb_view* csb, const uint32_t* group_bounds,
                             uint32_t ngroups, uint32_t tile_edge, uint32_t row_lo, uint32_t row_hi,
                             cieg_mat** out);
/* Single-pass SpMM on a row shard (the transposed-half
 * partials are reduce-scattered to the row owners): every stored tile of the
 * shard's rows is read once; y_dev (local rows) gets the row parts and the
 * transposed parts that land on owned rows, yhalo_dev (rows [lo, hi) of
 * cieg_matrix_partial_rows, m columns, ld m) the transposed partial sums for
 * rows owned by lower shards, which the caller sends to their owners and
 * adds there (dist.py partial_reduce: point to point, added in rank order).
 * x_dev as for cieg_spmm on a shard (globally addressed, halo rows backed).
 * On an unsharded matrix: cieg_spmm in single-pass mode (no partial rows).
 * Replaces the reference's fused-mode planner step (planner.cpp:116-122). */
int cieg_spmm_partial(cieg_ctx* ctx, const cieg_mat* mat, const double* x_dev, double* y_dev, uint32_t m,
                      double* yhalo_dev);
/* Rows [lo, hi) of the partials cieg_spmm_partial writes (hi = row_lo of the
 * shard; lo = hi when it has none). */
int cieg_matrix_partial_rows(const cieg_mat* mat, uint32_t* lo, uint32_t* hi);
/* Rows owned by a (shard) matrix: [row_lo, row_hi); the full matrix owns all. */
int cieg_matrix_rows(const cieg_mat* mat, uint32_t* row_lo, uint32_t* row_hi, uint32_t* halo_lo,
                     uint32_t* halo_hi);
/* Tile diagonal of the groups inside [row_lo, row_hi) (local row numbering). */
int cieg_precond_from_csb_range(cieg_ctx* ctx, const cieg_csb_view* csb, const uint32_t* group_bounds,
                                uint32_t ngroups, uint32_t row_lo, uint32_t row_hi, cieg_prec** out);
/* Run the context's work on a caller-owned stream (e.g. torch's current
 * stream) so it orders with the caller's collectives; NULL restores the
 * context's own stream. */
int cieg_ctx_set_stream(cieg_ctx* ctx, void* stream);

/* Collective hooks for the sharded solver (one process per GPU). */
typedef struct {
  void* user;
  /* in-place sum over ranks of `count` doubles in host memory (Gram partials) */
  int (*allreduce_sum)(void* user, double* host_buf, uint64_t count);
  /* gather before each SpMM: the rank's local rows of a row-distributed
   * block (device, local_rows x m) plus its neighbours' into x_full, a block
   * addressed with GLOBAL row indices (x_full + row * m) of which only the
   * shard's halo rows [halo_lo, halo_hi) (cieg_matrix_rows) are backed by
   * memory -- the only rows the shard's kernel reads. dist.py fills them by
   * a point-to-point halo exchange. */
  int (*allgather_rows)(void* user, const double* x_local_dev, uint32_t m, double* x_full_dev);
  /* optional (NULL: owner-computes shards). After a single-pass SpMM (the
   * SpMM mode's width rule, cieg_ctx_set_spmm_mode): send the transposed
   * partials for lower ranks' rows (yhalo_dev, rows [lo, hi) of
   * cieg_matrix_partial_rows, m columns) to their owners and add the ones
   * received into y_local_dev (local_rows x m) in ascending rank order --
   * the reduce-scatter of SURVEY.md 8(e), point to point. */
  int (*reduce_partials)(void* user, const double* yhalo_dev, uint32_t m, double* y_local_dev);
} cieg_dist_hooks;

/* The same collectives inside the library, on an NCCL communicator owned by
 * the context (libnccl.so.2 opened at run time): rank 0 creates the id,
 * the caller distributes it (e.g. torch.distributed), every rank inits its
 * context. cieg_lobpcg_solve_nccl then runs the sharded solve with the Gram
 * all-reduces on the device before the single D2H, the X halo exchange and
 * the single-pass partial reduction as grouped ncclSend/ncclRecv on the
 * context's stream (the planner's fused mode, planner.cpp:116-122). */
int cieg_nccl_unique_id(uint8_t* id_out /* 128 bytes */);
int cieg_ctx_nccl_init(cieg_ctx* ctx, const uint8_t* id /* 128 bytes */, int nranks, int rank);
int cieg_ctx_nccl_finalize(cieg_ctx* ctx);

/* ---- tall-skinny block kernels (proj/include/ci/block_vectors.hpp) ----- */
/* X^T Y (kx x ky, column major, written to out_host) -- ci::block_inner
 * (block_vectors.hpp:60, block_vectors.cpp:74-85). Partials are reduced in a
 * fixed order (deterministic). */
int cieg_block_inner(cieg_ctx* ctx, uint32_t n, const double* x_dev, uint32_t kx,
                     const double* y_dev, uint32_t ky, double* out_host);
/* out = Y G (G kin x kout column major, host) -- ci::linear_combination
 * (block_vectors.hpp:64, block_vectors.cpp:118-129). */
int cieg_linear_combination(cieg_ctx* ctx, uint32_t n, const double* y_dev, uint32_t kin,
                            const double* g_host, uint32_t kout, double* out_dev);
/* Y += X G -- ci::add_linear_combination (block_vectors.hpp:68,
 * block_vectors.cpp:139-160). */
int cieg_add_linear_combination(cieg_ctx* ctx, uint32_t n, double* y_dev, uint32_t ky,
                                const double* x_dev, uint32_t kx, const double* g_host);
/* Per-column Euclidean norms -- ci::column_norms (block_vectors.hpp:75). */
int cieg_column_norms(cieg_ctx* ctx, uint32_t n, const double* x_dev, uint32_t k,
                      double* out_host);

/* ---- tile-diagonal preconditioner (proj/include/ci/precond.hpp) -------- */
typedef struct {
  int inner_iters;             /* FOM iteration cap, 1..3 (precond.hpp:17) */
  int small_block_cutoff;      /* direct dense solve at or below (precond.hpp:18) */
  int engage_after;            /* precond.hpp:19 */
  double relres_gate;          /* precond.hpp:20 */
  double near_converged_factor;/* precond.hpp:21 (read by nothing, as in the reference) */
  double far_threshold;        /* precond.hpp:22 */
  double column_floor_factor;  /* precond.hpp:27 */
} cieg_precond_config;
/* Defaults of ci::PrecondConfig. */
void cieg_precond_config_default(cieg_precond_config* cfg);

/* Flattened ci::TileDiagonal (hamiltonian.hpp:58-63): ngroups contiguous
 * ranges [bounds[g], bounds[g+1]) covering [0, dim) and their dense blocks,
 * concatenated column-major (block g has (bounds[g+1]-bounds[g])^2 entries). */
typedef struct {
  uint32_t dim;
  uint32_t ngroups;
  const uint32_t* bounds;   /* ngroups + 1 */
  const double* blocks;     /* sum of n_g^2 */
} cieg_tilediag_view;
int cieg_precond_upload(cieg_ctx* ctx, const cieg_tilediag_view* tiles, cieg_prec** out);
/* Build the tile diagonal on the device from an uploaded H and a group
 * partition -- ci::extract_tile_diagonal (hamiltonian.cpp:178-203). */
int cieg_precond_from_csb(cieg_ctx* ctx, const cieg_csb_view* csb, const uint32_t* group_bounds,
                          uint32_t ngroups, cieg_prec** out);
int cieg_precond_destroy(cieg_prec* prec);

/* ci::choose_shifts (precond.hpp:47-48, precond.cpp:13-55), host scalar
 * logic. engage_out receives 0/1 per column. */
int cieg_choose_shifts(uint32_t k, const double* theta, const double* res_norm,
                       const double* x_norm, const double* relres, int iteration, double tol,
                       const cieg_precond_config* cfg, double* mu_out, int* engage_out);
/* W = apply_preconditioner(tiles, R, plan) -- ci::apply_preconditioner
 * (precond.hpp:53-54, precond.cpp:160-207); r_dev/w_dev row-major n x k. */
int cieg_precond_apply(cieg_ctx* ctx, const cieg_prec* prec, const double* r_dev, uint32_t k,
                       const double* mu_host, const int* engage_host,
                       const cieg_precond_config* cfg, double* w_dev);

/* ---- LOBPCG (proj/include/ci/lobpcg.hpp) ------------------------------- */
typedef struct {
  int k_want;          /* lobpcg.hpp:55 */
  double tol;          /* lobpcg.hpp:56 */
  int max_iter;        /* lobpcg.hpp:57 */
  cieg_precond_config precond_config; /* lobpcg.hpp:59 */
} cieg_lobpcg_options;
void cieg_lobpcg_options_default(cieg_lobpcg_options* opt);

/* Per-iteration observer (ci::IterationView, lobpcg.hpp:47-52). x_host is the
 * trial block (n x kt row-major) copied to the host only when an observer is
 * installed; pointers are valid during the call only. */
typedef void (*cieg_observer_fn)(void* user, int iteration, const double* x_host, uint32_t n,
                                 uint32_t kt, const double* theta, const double* relres);

/* ci::lobpcg_solve (lobpcg.hpp:67-68, lobpcg.cpp:216-387): X0 (host, n x kt
 * row-major) supplies the trial block; prec may be NULL (unpreconditioned).
 * Non-convergence is not an error: the report's converged flag is 0. */
int cieg_lobpcg_solve(cieg_ctx* ctx, const cieg_mat* mat, const double* x0_host, uint32_t kt,
                      const cieg_prec* prec, const cieg_lobpcg_options* opt,
                      cieg_observer_fn observer, void* observer_user, cieg_report** out);
/* Sharded ci::lobpcg_solve: mat from cieg_matrix_upload_shard, x0_host and
 * prec local to the rank's rows; every Gram is all-reduced and the SpMM input
 * all-gathered through `hooks`; identical control flow on every rank. The
 * report's trial vectors are the rank's local rows. */
int cieg_lobpcg_solve_dist(cieg_ctx* ctx, const cieg_mat* mat, const double* x0_host, uint32_t kt,
                           const cieg_prec* prec, const cieg_lobpcg_options* opt, const cieg_dist_hooks* hooks,
                           cieg_report** out);
/* The sharded solve with its collectives inside the library (the context's
 * NCCL communicator, cieg_ctx_nccl_init); same results as _dist. */
int cieg_lobpcg_solve_nccl(cieg_ctx* ctx, const cieg_mat* mat, const double* x0_host, uint32_t kt,
                           const cieg_prec* prec, const cieg_lobpcg_options* opt, cieg_report** out);
int cieg_report_destroy(cieg_report* rep);
/* SolveReport fields (lobpcg.hpp:34-43). */
int cieg_report_summary(const cieg_report* rep, int* converged, int* iterations,
                        double* norm_estimate, uint32_t* k_want, uint32_t* kt, uint64_t* history_rows);
/* counters: spmm_calls, spmv_equivalents, precond_applications, orthogonalizations. */
int cieg_report_counters(const cieg_report* rep, uint64_t* counters4);
int cieg_report_eigenvalues(const cieg_report* rep, double* out /* k_want */);
/* trial_vectors: n x kt row-major (eigenvectors are its first k_want columns). */
int cieg_report_trial_vectors(const cieg_report* rep, double* out);
/* history rows (iteration, column, relres, theta), in order. */
int cieg_report_history(const cieg_report* rep, int* iteration, int* column, double* relres,
                        double* theta);
/* Device-event time split of the solve in milliseconds:
 * [spmm, rayleigh_ritz, orthonormalization, preconditioner, residual, other, total]. */
int cieg_report_timing(const cieg_report* rep, double* ms7);

/* ---- lobpcg.hpp public helpers ------------------------------------------ */
/* ci::orthonormalize (lobpcg.hpp:92-93, lobpcg.cpp:89-119): y_dev (row-major
 * n x k, device) is projected against against_dev (n x ka, may be NULL) twice,
 * rank-revealing column selection at drop_tol, CholQR twice; the result is
 * written back packed (n x k_out, ld = k_out). */
int cieg_orthonormalize(cieg_ctx* ctx, double* y_dev, uint32_t n, uint32_t k, double drop_tol,
                        const double* against_dev, uint32_t ka, uint32_t* k_out);
/* ci::rayleigh_ritz (lobpcg.hpp:84-86, lobpcg.cpp:121-145) on an orthonormal
 * basis Y and HY (device, n x m row-major): theta_out[k_trial], g_out
 * (m x k_trial column-major). CIEG_ERR_INDEFINITE when Y^T Y deviates from I
 * by more than 1e-6. */
int cieg_rayleigh_ritz(cieg_ctx* ctx, const double* y_dev, const double* hy_dev, uint32_t n, uint32_t m,
                       uint32_t k_trial, double* theta_out, double* g_out);
/* ci::residual_norms (lobpcg.hpp:97-99, lobpcg.cpp:147-169): relative
 * residuals |H x_j - theta_j x_j| / max(est |x_j|, 1e-300); norm_est <= 0
 * means "none" (est = max |theta|). x_dev device n x k row-major. */
int cieg_residual_norms(cieg_ctx* ctx, const cieg_mat* mat, const double* x_dev, uint32_t k, const double* theta,
                        double norm_est, double* out);

/* ---- starting blocks (proj/include/ci/guess.hpp) ----------------------- */
/* Leading principal block H[0:dim, 0:dim] of an uploaded matrix as a matrix
 * of its own, sharing the parent's device tile stream (valid while the
 * parent lives); dim must end on a device panel boundary (e.g. a sector or
 * group boundary). The truncated-space problems of multilevel_guess. */
int cieg_matrix_leading_view(cieg_ctx* ctx, const cieg_mat* mat, uint32_t dim, cieg_mat** out);
/* ci::pad_from_subspace (guess.hpp:21, guess.cpp:14-23), host buffers. */
int cieg_pad_from_subspace(const double* x_host, uint32_t n1, uint32_t k, uint32_t dim, double* out_host);
typedef struct {
  int k_want;    /* guess.hpp:49 */
  int k_trial;   /* guess.hpp:50 */
  double tol;    /* guess.hpp:51 */
  int max_iter;  /* guess.hpp:52 */
  uint64_t seed; /* guess.hpp:53 */
} cieg_multilevel_options;
void cieg_multilevel_options_default(cieg_multilevel_options* opt);
typedef struct { /* ci::LevelReport (guess.hpp:31-37); nmax -> the level dimension */
  uint32_t dim;
  int iterations;
  int converged;
  double seconds;
} cieg_level_report;
/* ci::multilevel_guess (guess.hpp:60-62, guess.cpp:66-117): level_dims[0..nlevels)
 * are the ascending truncated dimensions (leading blocks, reference levels =
 * nlevels + 1); unpreconditioned LOBPCG per level, random start at the
 * smallest. guess_host: n x k_trial row-major capacity, k_out = its width
 * (packed); levels_out[nlevels]. */
int cieg_multilevel_guess(cieg_ctx* ctx, const cieg_mat* mat, const uint32_t* level_dims, uint32_t nlevels,
                          const cieg_multilevel_options* opt, double* guess_host, uint32_t* k_out,
                          cieg_level_report* levels_out);

/* ---- Lanczos baseline (proj/include/ci/lanczos.hpp) -------------------- */
/* Checkpoint hook (LanczosOptions::observer, lanczos.hpp:18-21): step count,
 * the tridiagonal coefficients alpha[0..m) / beta[0..m), and the Lanczos
 * basis (column-major n x m) copied to the host only when an observer is
 * installed; pointers are valid during the call only. */
typedef void (*cieg_lanczos_observer_fn)(void* user, int m, const double* alpha, const double* beta,
                                         const double* basis_host, uint32_t n);
typedef struct {
  int k_want;   /* lanczos.hpp:15 */
  double tol;   /* lanczos.hpp:16 */
  int max_iter; /* lanczos.hpp:17 */
  cieg_lanczos_observer_fn observer;
  void* observer_user;
} cieg_lanczos_options;
void cieg_lanczos_options_default(cieg_lanczos_options* opt);
/* ci::lanczos_checkpoint (lanczos.hpp:26, lanczos.cpp:11-15): 1 on the
 * staggered grid (every 10 steps to 100, 20 to 200, then 40). */
int cieg_lanczos_checkpoint(int m);
/* ci::lanczos_default_start (lanczos.hpp:30, lanczos.cpp:17-22) given the end
 * of the lowest stratum: ones on [0, stratum_end), normalised; out: n doubles. */
int cieg_lanczos_default_start(uint32_t n, uint32_t stratum_end, double* out);
/* ci::lanczos_solve (lanczos.hpp:35-36, lanczos.cpp:24-136): v0 host vector
 * of length n. Same report schema as cieg_lobpcg_solve (k_want = kt = the
 * number of Ritz pairs returned; counters: spmm_calls, spmv_equivalents, 0,
 * orthogonalizations; timing: spmm, ritz analysis, reorthogonalisation,
 * 0, 0, other, total). */
int cieg_lanczos_solve(cieg_ctx* ctx, const cieg_mat* mat, const double* v0_host, const cieg_lanczos_options* opt,
                       cieg_report** out);

/* ---- synthetic sector generator (BASELINE.json configs) ---------------- */
/* Deterministic sector/tile matrix of SURVEY.md 8(d): ns equal sectors,
 * tile grid restarting at every sector, tiles kept for |ds| <= band with
 * probability p (diagonal tiles always), entries with probability q, values
 * N(0,1)/sqrt(avg full-row nnz) (Box-Muller over hash3 streams, proj/include/
 * ci/rng.hpp), diagonal 10 s + U(-2,2). Produces a host CSB (beta-bounded,
 * sector-aligned blocks) and its group (= tile) partition. */
typedef struct {
  uint32_t n;
  uint32_t sectors;
  uint32_t tile;      /* tile edge T */
  uint32_t band;      /* |s_a - s_b| <= band (2) */
  double p;           /* tile keep probability */
  double q;           /* entry probability inside a kept tile */
  uint64_t seed;
  int precision;      /* 0 single, 1 double */
  uint32_t beta;      /* CSB block bound (< 2^16) */
} cieg_gen_params;
/* Expected stored nnz (lower incl. diagonal) for the parameters. */
double cieg_gen_expected_nnz(const cieg_gen_params* prm);
/* Expected full-row off-diagonal count used for the value scale. */
double cieg_gen_avg_row_nnz(const cieg_gen_params* prm);
/* Exact stored-entry count of the generated matrix (0 on bad parameters). */
uint64_t cieg_gen_count_nnz(const cieg_gen_params* prm);
int cieg_generate_csb(const cieg_gen_params* prm, cieg_host_csb** out);
int cieg_host_csb_destroy(cieg_host_csb* h);
/* Borrowed views into the generated matrix (valid until destroy). */
int cieg_host_csb_view(const cieg_host_csb* h, cieg_csb_view* view, uint64_t* nnz);
int cieg_host_csb_groups(const cieg_host_csb* h, const uint32_t** bounds, uint32_t* ngroups);

/* The same generator run on the GPU, writing the device tile stream directly
 * (no host CSB; bit-identical tile stream to cieg_matrix_upload of
 * cieg_generate_csb). Owner rows [row_lo, row_hi) (0, 0 = all) for a shard;
 * tile_edge 0 = choose. SURVEY.md 8(f) rank 1. */
/* The device panel grid cieg_generate_device plans for these parameters
 * (panel_start[npanels + 1]; panel_start = NULL returns the count): shard
 * row ranges must be unions of whole panels. */
int cieg_generated_panels(const cieg_gen_params* prm, uint32_t tile_edge, uint32_t* panel_start, uint32_t cap,
                          uint32_t* npanels);
int cieg_generate_device(cieg_ctx* ctx, const cieg_gen_params* prm, uint32_t tile_edge, uint32_t row_lo,
                         uint32_t row_hi, cieg_mat** out);
/* Tile-diagonal preconditioner built on the device from the matrix's own
 * diagonal tiles (groups = generator tiles) -- ci::extract_tile_diagonal
 * (hamiltonian.cpp:178-203) without a host TileDiagonal; shard-local. */
int cieg_precond_from_matrix(cieg_ctx* ctx, const cieg_mat* mat, cieg_prec** out);
/* Borrowed group partition of a matrix (ngroups + 1 bounds; 0 groups when unknown). */
int cieg_matrix_groups(const cieg_mat* mat, const uint32_t** bounds, uint32_t* ngroups);
/* Copy the device tile stream to the host (tile_off: ntiles + 1; tile_pi/pj:
 * ntiles; idx/val: tile_off[ntiles] slots); any pointer may be NULL. */
int cieg_matrix_export(const cieg_mat* mat, uint64_t* tile_off, uint32_t* tile_pi, uint32_t* tile_pj,
                       uint32_t* idx, void* val);

/* ci::random_block (block_vectors.cpp:162-174): out n x k row-major,
 * entries 2*unit(hash3(seed, i, j)) - 1. */
int cieg_random_block(uint32_t n, uint32_t k, uint64_t seed, double* out_host);
/* Rows [row_lo, row_hi) of the same block (a shard's rows of X0). */
int cieg_random_block_rows(uint32_t row_lo, uint32_t row_hi, uint32_t k, uint64_t seed, double* out_host);

#ifdef __cplusplus
}
#endif
#endif /* CIEG_H */
