// context.hpp -- device-side objects behind the opaque C handles.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <deque>
#include <vector>

#include "cieg_internal.hpp"

namespace cieg {

inline void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) fail(CIEG_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}
#define CIEG_CUDA(call) ::cieg::cuda_check((call), #call)

// Growable device scratch buffer.
struct DevBuf {
  void* ptr = nullptr;
  std::size_t bytes = 0;
  void* get(std::size_t want) {
    if (want > bytes) {
      if (ptr) cudaFree(ptr);
      ptr = nullptr;
      bytes = 0;
      CIEG_CUDA(cudaMalloc(&ptr, want));
      bytes = want;
    }
    return ptr;
  }
  void release() {
    if (ptr) cudaFree(ptr);
    ptr = nullptr;
    bytes = 0;
  }
};

struct PinnedBuf {
  void* ptr = nullptr;
  std::size_t bytes = 0;
  void* get(std::size_t want) {
    if (want > bytes) {
      if (ptr) cudaFreeHost(ptr);
      ptr = nullptr;
      bytes = 0;
      CIEG_CUDA(cudaMallocHost(&ptr, want));
      bytes = want;
    }
    return ptr;
  }
  void release() {
    if (ptr) cudaFreeHost(ptr);
    ptr = nullptr;
    bytes = 0;
  }
};

struct SlicedPlan;  // spmm_i8.cu
struct HostCopier;  // capi.cu: the helper thread that copies finished downloads out of the pinned ring
struct NcclPlane;   // nccl_plane.cu

}  // namespace cieg

struct cieg_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;      // stream all work is enqueued on
  cudaStream_t own_stream = nullptr;  // the context's own stream
  std::uint64_t launches = 0;
  int exact_order = 0;
  int spmm_mode = -1;  // CIEG_SPMM_*; -1 = not set (CIEG_SPMM_MODE env, else auto)  // 1: K5 reproduces the reference's operation order bit for bit
  int sm_count = 148;
  cieg::DevBuf scratch_x, scratch_y, scratch_red, scratch_small;
  cieg::DevBuf scratch_x2, scratch_y2, scratch_x3, scratch_y3;  // ring buffers of the pipelined host batch
  cieg::DevBuf scratch_flag;            // K1 non-finite-input flag
  cieg::DevBuf scratch_partial;         // single-pass K1: transposed partial products
  unsigned spmm_launch_id = 0;          // tags the flag per K1 launch
  std::deque<cieg::DevBuf> solver_pool; // LOBPCG work blocks, reused across solves
  cieg::PinnedBuf pinned_small;
  cieg::PinnedBuf pinned_stage;         // pageable host X/U: chunked staging ring (capi.cu)
  cudaEvent_t stage_ev[4] = {};
  // the chunk-pipelined host SpMM (spmm_i8.cu sliced_spmm_host): copy streams, the download ring, an event pool
  cudaStream_t pipe_up = nullptr, pipe_down = nullptr;
  cieg::PinnedBuf pinned_stage_down;
  std::vector<cudaEvent_t> pipe_ev;
  cieg::HostCopier* copier = nullptr;
  // phase timers (report.hpp Clock): event pairs read at the end of a solve,
  // so timing a phase does not synchronise the host with the device
  struct ClockRec {
    cudaEvent_t a, b;
    double* slot;
  };
  std::vector<cudaEvent_t> ev_pool;
  std::vector<ClockRec> ev_pending;
  cieg::NcclPlane* nccl = nullptr;      // communicator of a sharded solve (cieg_ctx_nccl_init)
  bool nccl_grams = false;              // Grams all-reduced on the device inside gram()/combine_gram()
};

struct cieg_mat {
  cieg_ctx* ctx = nullptr;
  std::uint32_t dim = 0;
  std::uint32_t tile_edge = 0;
  int precision = 0;
  std::uint64_t nnz = 0;
  std::uint32_t npanels = 0;
  std::uint64_t ntiles = 0;
  std::uint64_t tile_bytes = 0;
  std::vector<std::uint32_t> panel_start_host;
  std::vector<std::uint32_t> group_bounds_host;  // group (= tile) partition, when known
  std::vector<std::uint32_t> tile_pi_host, tile_pj_host;
  std::vector<std::uint64_t> tile_off_host;
  // device arrays
  std::uint32_t* panel_start = nullptr;
  std::uint64_t* tile_off = nullptr;
  std::uint32_t* idx = nullptr;
  void* val = nullptr;
  std::uint32_t* work_off = nullptr;
  std::uint32_t* work_tile = nullptr;
  std::uint32_t* work_other = nullptr;
  std::uint32_t* work_kind = nullptr;
  std::uint32_t row_lo = 0, row_hi = 0, halo_lo = 0, halo_hi = 0;  // owner rows / X rows read
  std::uint32_t sched_ctas = 0;
  std::uint32_t* sched_off = nullptr;
  std::uint32_t* sched = nullptr;
  // single-pass schedule (full matrices; tiling.hpp): one item per stored tile
  std::uint32_t sp_ctas = 0, sp_items = 0;
  std::uint32_t* sp_sched_off = nullptr;
  std::uint32_t* sp_sched = nullptr;
  std::uint32_t* sp_col_off = nullptr;
  std::uint32_t* sp_col_items = nullptr;
  std::uint32_t sp_partial_lo = 0;  // shards: partial rows [sp_partial_lo, row_lo) for lower shards
  // a leading-block view (cieg_matrix_leading_view) borrows panel_start,
  // tile_off, idx and val from its parent and owns only its work lists
  bool borrowed_stream = false;
  // integer-slice tensor-core K1 (spmm_i8.cu): digit records, built on first use
  cieg::SlicedPlan* sliced = nullptr;
  ~cieg_mat();
};

namespace cieg {

// Bank-aware ordering of the entries inside every tile (reorder.cu); run
// once on every freshly built device tile stream.
void order_tile_entries(cieg_ctx* ctx, cieg_mat* m);

// The SpMM mode's rule for block width mc on a matrix with a single-pass
// schedule (auto: single pass for mc <= 8); single_pass_default adds, in
// auto mode, the memory check of single_pass_fits.
bool single_pass_rule(const cieg_ctx* ctx, const cieg_mat* m, std::uint32_t mc);
bool single_pass_default(const cieg_ctx* ctx, const cieg_mat* m, std::uint32_t mc);
// The per-tile partial slots of a single pass at width mc take at most a
// quarter of the free device memory (or are already allocated).
bool single_pass_fits(const cieg_ctx* ctx, const cieg_mat* m, std::uint32_t mc);
constexpr std::uint32_t kSinglePassMaxCols = 8;

// Upload the work lists and both K1 schedules of a tiling.
struct HostTiles;
void upload_schedule(cieg_mat* m, const HostTiles& ht);

// Launch the owner-computes SpMM over device X/Y (row-major, ld = ldx/ldy).
// On a shard, shard_single_pass selects the single pass; yhalo receives
// the transposed partials for rows [sp_partial_lo, row_lo) (ld ldh; may be
// null when the shard has no such rows).
void launch_spmm(cieg_ctx* ctx, const cieg_mat* m, const double* x, std::uint32_t ldx, double* y,
                 std::uint32_t ldy, std::uint32_t mcols, double* yhalo = nullptr, std::uint32_t ldh = 0,
                 bool shard_single_pass = false);

// Integer-slice (Ozaki) K1 on tcgen05 (spmm_i8.cu): fp32 H, 128-row panels,
// full (unsharded) matrices with a single-pass schedule.
bool sliced_supported(const cieg_mat* m);
// builds the slice records on first use; false when unsupported or H holds Inf/NaN
bool sliced_ready(cieg_ctx* ctx, cieg_mat* m);
// the mode's choice for width mc (auto: sliced for mc >= kSlicedMinCols)
bool sliced_rule(const cieg_ctx* ctx, const cieg_mat* m, std::uint32_t mc);
constexpr std::uint32_t kSlicedMinCols = 2;  // config 2, sliced vs the DMMA / scalar single pass: m = 1 2.37 vs 2.10 ms; m = 4 2.41 vs 2.79; m = 8 2.43 vs 2.95; m = 16 2.59 vs 4.95
// Digitize X and run the sliced kernel: every row of Y written (row parts and
// transposed parts accumulated in exact fixed point, then converted); the
// caller runs the tiny-entry and non-finite fix-ups.
void launch_spmm_sliced(cieg_ctx* ctx, cieg_mat* m, const double* x, std::uint32_t ldx, double* y,
                        std::uint32_t ldy, std::uint32_t mc, unsigned* nonfinite, unsigned launch_id);
void destroy_sliced(cieg_mat* m);
// ci::spmm's host call on the sliced kernel, pipelined over row chunks (upload,
// kernels and download overlap); false when the sliced kernel does not apply
// (the caller then runs upload -> launch_spmm -> download).
bool sliced_spmm_host(cieg_ctx* ctx, cieg_mat* m, const double* x_host, double* y_host, std::uint32_t mc,
                      bool x_pinned, bool y_pinned);
// Host side of pageable buffers (capi.cu). host_copy_in: threaded copy into a
// pinned upload slot on the calling thread (`shared`: the helper thread is
// copying too -- half the threads each). copier_submit: once `ev` completes,
// the helper thread copies a finished download out of its ring slot
// (non-temporal stores); returns the number of jobs submitted so far.
// copier_wait blocks until that many jobs are done (throws on a failed one);
// copier_drain waits for all of them and never throws.
void host_copy_in(void* dst, const void* src, std::size_t bytes, bool shared);
std::size_t copier_submit(cieg_ctx* ctx, cudaEvent_t ev, void* dst, const void* src, std::size_t bytes);
std::size_t copier_submitted(cieg_ctx* ctx);
void copier_wait(cieg_ctx* ctx, std::size_t jobs);
void copier_drain(cieg_ctx* ctx) noexcept;
void destroy_copier(cieg_ctx* ctx);
// K1's non-finite-input flag and the fix-up of the launch tagged launch_id
unsigned* nonfinite_flag(cieg_ctx* ctx);
void launch_nonfinite_fix(cieg_ctx* ctx, const cieg_mat* m, const double* x, std::uint32_t ldx, double* y,
                          std::uint32_t ldy, std::uint32_t mc, unsigned launch_id);
// the K1 mode launch_spmm runs for width mc (CIEG_SPMM_OWNER / SINGLE_PASS / SLICED)
int spmm_effective_mode(cieg_ctx* ctx, cieg_mat* m, std::uint32_t mc);
// NCCL data plane (nccl_plane.cu)
struct NcclSolve;
bool nccl_active(const cieg_ctx* ctx);
void nccl_allreduce_sum(cieg_ctx* ctx, double* dev, std::size_t count);
void destroy_nccl(cieg_ctx* ctx);
NcclSolve* nccl_solve_begin(cieg_ctx* ctx, const cieg_mat* mat);
void nccl_solve_end(NcclSolve* s);
int nccl_hook_allreduce(void* user, double* host_buf, std::uint64_t count);
int nccl_hook_gather(void* user, const double* x_local, std::uint32_t m, double* full);
int nccl_hook_reduce_partials(void* user, const double* yhalo, std::uint32_t m, double* y_local);
// fp64 terms of the stored entries too small to slice exactly (after sp_reduce)
void launch_sliced_tiny_fix(cieg_ctx* ctx, const cieg_mat* m, const double* x, std::uint32_t ldx, double* y,
                            std::uint32_t ldy, std::uint32_t mc);

}  // namespace cieg
