// capi.cu -- C ABI plumbing: errors, contexts, matrix upload, SpMM entry
// points (include/cieg.h).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#if defined(__SSE2__)
#include <emmintrin.h>
#endif
#include <condition_variable>
#include <deque>
#include <memory>
#include <mutex>
#include <thread>
#include <omp.h>
#include <string>

#include "context.hpp"
#include "tiling.hpp"

namespace cieg {

namespace {
thread_local std::string g_last_error;
}
void set_last_error(const std::string& msg) { g_last_error = msg; }
void clear_last_error() { g_last_error.clear(); }

template <typename T>
T* upload_vec(const std::vector<T>& v) {
  if (v.empty()) return nullptr;
  T* d = nullptr;
  CIEG_CUDA(cudaMalloc(&d, v.size() * sizeof(T)));
  CIEG_CUDA(cudaMemcpy(d, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice));
  return d;
}

}  // namespace cieg

cieg_mat::~cieg_mat() {
  cieg::destroy_sliced(this);
  if (!borrowed_stream) {
    cudaFree(panel_start);
    cudaFree(tile_off);
    cudaFree(idx);
    cudaFree(val);
  }
  cudaFree(sp_sched_off);
  cudaFree(sp_sched);
  cudaFree(sp_col_off);
  cudaFree(sp_col_items);
  cudaFree(work_off);
  cudaFree(work_tile);
  cudaFree(work_other);
  cudaFree(work_kind);
  cudaFree(sched_off);
  cudaFree(sched);
}

namespace {

__global__ void count_real_kernel(const std::uint32_t* idx, std::uint64_t n, std::uint32_t sentinel,
                                  unsigned long long* count) {
  unsigned long long c = 0;
  for (std::uint64_t i = blockIdx.x * std::uint64_t(blockDim.x) + threadIdx.x; i < n;
       i += std::uint64_t(gridDim.x) * blockDim.x)
    c += idx[i] != sentinel;
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0) atomicAdd(count, c);
}

// Real (non-padding) entries among the first n slots of a tile stream.
std::uint64_t count_real_entries(cieg_ctx* ctx, const std::uint32_t* idx, std::uint64_t n, std::uint32_t sentinel) {
  if (n == 0) return 0;
  unsigned long long* d = nullptr;
  CIEG_CUDA(cudaMalloc(&d, sizeof(unsigned long long)));
  unsigned long long h = 0;
  CIEG_CUDA(cudaMemsetAsync(d, 0, sizeof h, ctx->stream));
  count_real_kernel<<<4 * ctx->sm_count, 256, 0, ctx->stream>>>(idx, n, sentinel, d);
  ++ctx->launches;
  CIEG_CUDA(cudaMemcpyAsync(&h, d, sizeof h, cudaMemcpyDeviceToHost, ctx->stream));
  CIEG_CUDA(cudaStreamSynchronize(ctx->stream));
  cudaFree(d);
  return h;
}

}  // namespace

extern "C" {

const char* cieg_last_error(void) { return cieg::g_last_error.c_str(); }
const char* cieg_version(void) { return "cieg 0.1 (sm_100a)"; }

int cieg_device_alloc(cieg_ctx* ctx, uint64_t bytes, void** out) {
  return cieg::guarded([&] {
    if (!ctx || !out) cieg::fail(CIEG_ERR_ARGUMENT, "cieg_device_alloc: null argument");
    CIEG_CUDA(cudaSetDevice(ctx->device));
    *out = nullptr;
    CIEG_CUDA(cudaMalloc(out, std::max<uint64_t>(1, bytes)));
  });
}

int cieg_device_free(cieg_ctx* ctx, void* p) {
  return cieg::guarded([&] {
    if (!ctx) cieg::fail(CIEG_ERR_ARGUMENT, "cieg_device_free: null context");
    CIEG_CUDA(cudaSetDevice(ctx->device));
    if (p) CIEG_CUDA(cudaFree(p));
  });
}

int cieg_memcpy(cieg_ctx* ctx, void* dst, const void* src, uint64_t bytes, int kind) {
  return cieg::guarded([&] {
    if (!ctx || (bytes && (!dst || !src))) cieg::fail(CIEG_ERR_ARGUMENT, "cieg_memcpy: null argument");
    static const cudaMemcpyKind kinds[3] = {cudaMemcpyHostToDevice, cudaMemcpyDeviceToHost, cudaMemcpyDeviceToDevice};
    if (kind < 0 || kind > 2) cieg::fail(CIEG_ERR_ARGUMENT, "cieg_memcpy: kind must be 0 (H2D), 1 (D2H) or 2 (D2D)");
    CIEG_CUDA(cudaSetDevice(ctx->device));
    if (bytes) CIEG_CUDA(cudaMemcpyAsync(dst, src, bytes, kinds[kind], ctx->stream));
    CIEG_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

int cieg_ctx_create(int device, cieg_ctx** out) {
  return cieg::guarded([&] {
    if (!out) cieg::fail(CIEG_ERR_ARGUMENT, "cieg_ctx_create: null output");
    int n = 0;
    CIEG_CUDA(cudaGetDeviceCount(&n));
    if (device < 0 || device >= n) cieg::fail(CIEG_ERR_ARGUMENT, "cieg_ctx_create: bad device index");
    CIEG_CUDA(cudaSetDevice(device));
    auto* c = new cieg_ctx;
    c->device = device;
    cudaDeviceProp prop;
    CIEG_CUDA(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10)
      cieg::fail(CIEG_ERR_CUDA, std::string("libcieg is built for sm_100a; device is ") + prop.name);
    c->sm_count = prop.multiProcessorCount;
    CIEG_CUDA(cudaStreamCreateWithFlags(&c->own_stream, cudaStreamNonBlocking));
    c->stream = c->own_stream;
    *out = c;
  });
}

int cieg_ctx_destroy(cieg_ctx* ctx) {
  if (!ctx) return CIEG_OK;
  cudaSetDevice(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  ctx->scratch_x.release();
  ctx->scratch_y.release();
  ctx->scratch_x2.release();
  ctx->scratch_y2.release();
  ctx->scratch_x3.release();
  ctx->scratch_y3.release();
  ctx->scratch_red.release();
  ctx->scratch_small.release();
  ctx->scratch_flag.release();
  ctx->scratch_partial.release();
  for (auto& b : ctx->solver_pool) b.release();
  ctx->pinned_small.release();
  ctx->pinned_stage.release();
  ctx->pinned_stage_down.release();
  for (auto& e : ctx->pipe_ev) cudaEventDestroy(e);
  if (ctx->pipe_up) cudaStreamDestroy(ctx->pipe_up);
  if (ctx->pipe_down) cudaStreamDestroy(ctx->pipe_down);
  cieg::destroy_copier(ctx);
  cieg::destroy_nccl(ctx);
  for (auto& e : ctx->stage_ev)
    if (e) cudaEventDestroy(e);
  for (auto& r : ctx->ev_pending) {
    cudaEventDestroy(r.a);
    cudaEventDestroy(r.b);
  }
  for (auto e : ctx->ev_pool) cudaEventDestroy(e);
  cudaStreamSynchronize(ctx->own_stream);
  cudaStreamDestroy(ctx->own_stream);
  delete ctx;
  return CIEG_OK;
}

int cieg_ctx_synchronize(cieg_ctx* ctx) {
  return cieg::guarded([&] {
    if (!ctx) cieg::fail(CIEG_ERR_ARGUMENT, "null context");
    CIEG_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

void* cieg_ctx_stream(cieg_ctx* ctx) { return ctx ? static_cast<void*>(ctx->stream) : nullptr; }
uint64_t cieg_ctx_launch_count(const cieg_ctx* ctx) { return ctx ? ctx->launches : 0; }

}  // extern "C"

namespace {

std::uint32_t choose_tile_edge(const cieg_csb_view* csb, const uint32_t* group_bounds, uint32_t ngroups,
                               uint32_t tile_edge) {
  std::uint32_t te = tile_edge;
  if (te == 0) {
    // Tile edge follows the group size: 64-row groups -> 64, else 128.
    te = 128;
    if (group_bounds && ngroups > 0) {
      std::uint32_t mx = 0;
      for (std::uint32_t g = 0; g < ngroups; ++g) mx = std::max(mx, group_bounds[g + 1] - group_bounds[g]);
      if (mx <= 64) te = 64;
    }
  }
  if (te != 64 && te != 128) cieg::fail(CIEG_ERR_CONFIG, "tile edge must be 64 or 128");
  if (csb->precision == 1) te = 64;  // fp64 dense tiles: 64 rows keep two buffers in shared memory
  return te;
}

}  // namespace

namespace cieg {
void upload_schedule(cieg_mat* m, const HostTiles& ht) {
  m->work_off = upload_vec(ht.work_off);
  m->work_tile = upload_vec(ht.work_tile);
  m->work_other = upload_vec(ht.work_other);
  m->work_kind = upload_vec(ht.work_kind);
  m->sched_ctas = static_cast<std::uint32_t>(ht.sched_off.size() - 1);
  m->sched_off = upload_vec(ht.sched_off);
  m->sched = upload_vec(ht.sched);
  if (!ht.sp_sched_off.empty()) {
    m->sp_ctas = static_cast<std::uint32_t>(ht.sp_sched_off.size() - 1);
    m->sp_items = static_cast<std::uint32_t>(ht.sp_sched.size() / 8);
    m->sp_sched_off = upload_vec(ht.sp_sched_off);
    m->sp_sched = upload_vec(ht.sp_sched);
    m->sp_col_off = upload_vec(ht.sp_col_off);
    m->sp_col_items = upload_vec(ht.sp_col_items);
  }
  m->sp_partial_lo = ht.sp_partial_lo;
}
}  // namespace cieg

namespace {

cieg_mat* upload_tiles(cieg_ctx* ctx, cieg::HostTiles& ht) {
  cieg::build_schedule(ht, static_cast<std::uint32_t>(ctx->sm_count));
  auto* m = new cieg_mat;
  try {
    m->ctx = ctx;
    m->dim = ht.dim;
    m->tile_edge = ht.tile_edge;
    m->precision = ht.precision;
    m->nnz = ht.nnz;
    m->npanels = ht.npanels();
    m->ntiles = ht.ntiles();
    m->row_lo = ht.row_lo;
    m->row_hi = ht.row_hi;
    m->halo_lo = ht.halo_lo;
    m->halo_hi = ht.halo_hi;
    m->panel_start_host = ht.panel_start;
    m->tile_pi_host = ht.tile_pi;
    m->tile_pj_host = ht.tile_pj;
    m->tile_off_host = ht.tile_off;
    m->panel_start = cieg::upload_vec(ht.panel_start);
    m->tile_off = cieg::upload_vec(ht.tile_off);
    m->idx = cieg::upload_vec(ht.idx);
    if (ht.precision == 0)
      m->val = cieg::upload_vec(ht.val32);
    else
      m->val = cieg::upload_vec(ht.val64);
    cieg::upload_schedule(m, ht);
    m->tile_bytes = ht.tile_off.back() * (4 + (ht.precision == 0 ? 4 : 8));
    cieg::order_tile_entries(ctx, m);
  } catch (...) {
    delete m;
    throw;
  }
  return m;
}

}  // namespace

extern "C" {

int cieg_matrix_upload(cieg_ctx* ctx, const cieg_csb_view* csb, const uint32_t* group_bounds,
                       uint32_t ngroups, uint32_t tile_edge, cieg_mat** out) {
  return cieg_matrix_upload_cuts(ctx, csb, group_bounds, ngroups, tile_edge, nullptr, 0, out);
}

int cieg_matrix_upload_cuts(cieg_ctx* ctx, const cieg_csb_view* csb, const uint32_t* group_bounds,
                            uint32_t ngroups, uint32_t tile_edge, const uint32_t* cuts, uint32_t ncuts,
                            cieg_mat** out) {
  return cieg::guarded([&] {
    if (!ctx || !csb || !out || (ncuts && !cuts)) cieg::fail(CIEG_ERR_ARGUMENT, "cieg_matrix_upload: null argument");
    if (csb->precision != 0 && csb->precision != 1) cieg::fail(CIEG_ERR_FORMAT, "bad precision tag");
    CIEG_CUDA(cudaSetDevice(ctx->device));
    const std::uint32_t te = choose_tile_edge(csb, group_bounds, ngroups, tile_edge);
    std::vector<std::uint32_t> panels = cieg::plan_panels(csb->dim, group_bounds, ngroups, te, cuts, ncuts);
    cieg::HostTiles ht;
    cieg::build_tiles(*csb, panels, te, ht);
    *out = upload_tiles(ctx, ht);
    if (group_bounds && ngroups) (*out)->group_bounds_host.assign(group_bounds, group_bounds + ngroups + 1);
  });
}

int cieg_matrix_leading_view(cieg_ctx* ctx, const cieg_mat* m, uint32_t dim, cieg_mat** out) {
  return cieg::guarded([&] {
    if (!ctx || !m || !out) cieg::fail(CIEG_ERR_ARGUMENT, "cieg_matrix_leading_view: null argument");
    if (m->row_lo != 0 || m->row_hi != m->dim) cieg::fail(CIEG_ERR_CONFIG, "leading view of a shard");
    if (m->tile_pi_host.empty() && m->ntiles) cieg::fail(CIEG_ERR_CONFIG, "matrix keeps no host tile map");
    const std::vector<std::uint32_t>& ps = m->panel_start_host;
    const auto pit = std::lower_bound(ps.begin(), ps.end(), dim);
    if (dim == 0 || dim > m->dim || pit == ps.end() || *pit != dim)
      cieg::fail(CIEG_ERR_DIMENSION, "leading block must end on a panel boundary inside the matrix");
    const std::uint32_t pd = static_cast<std::uint32_t>(pit - ps.begin());
    // tiles are sorted by (pi, pj): those inside [0, dim)^2 are a prefix
    const std::uint64_t td = static_cast<std::uint64_t>(
        std::lower_bound(m->tile_pi_host.begin(), m->tile_pi_host.end(), pd) - m->tile_pi_host.begin());
    cieg::HostTiles ht;
    ht.dim = dim;
    ht.tile_edge = m->tile_edge;
    ht.precision = m->precision;
    ht.panel_start.assign(ps.begin(), ps.begin() + pd + 1);
    ht.tile_pi.assign(m->tile_pi_host.begin(), m->tile_pi_host.begin() + td);
    ht.tile_pj.assign(m->tile_pj_host.begin(), m->tile_pj_host.begin() + td);
    ht.tile_off.assign(m->tile_off_host.begin(), m->tile_off_host.begin() + td + 1);
    ht.row_lo = ht.halo_lo = 0;
    ht.row_hi = ht.halo_hi = dim;
    cieg::build_work_lists(ht, 0, pd);
    cieg::build_schedule(ht, static_cast<std::uint32_t>(ctx->sm_count));
    CIEG_CUDA(cudaSetDevice(ctx->device));
    auto v = std::make_unique<cieg_mat>();
    v->borrowed_stream = true;
    v->ctx = ctx;
    v->dim = dim;
    v->tile_edge = m->tile_edge;
    v->precision = m->precision;
    v->npanels = pd;
    v->ntiles = td;
    v->row_lo = v->halo_lo = 0;
    v->row_hi = v->halo_hi = dim;
    v->panel_start_host = ht.panel_start;
    v->tile_pi_host = ht.tile_pi;
    v->tile_pj_host = ht.tile_pj;
    v->tile_off_host = ht.tile_off;
    for (std::uint32_t b : m->group_bounds_host)
      if (b <= dim) v->group_bounds_host.push_back(b);
    v->panel_start = m->panel_start;
    v->tile_off = m->tile_off;
    v->idx = m->idx;
    v->val = m->val;
    cieg::upload_schedule(v.get(), ht);
    // stored entries of the block (padding sentinels excluded), for info()
    v->nnz = count_real_entries(ctx, m->idx, ht.tile_off.back(), m->tile_edge | (m->tile_edge << 16));
    v->tile_bytes = ht.tile_off.back() * (4 + (m->precision == 0 ? 4 : 8));
    *out = v.release();
  });
}

int cieg_matrix_upload_shard(cieg_ctx* ctx, const cieg_csb_view* csb, const uint32_t* group_bounds,
                             uint32_t ngroups, uint32_t tile_edge, uint32_t row_lo, uint32_t row_hi,
                             cieg_mat** out) {
  return cieg::guarded([&] {
    if (!ctx || !csb || !out) cieg::fail(CIEG_ERR_ARGUMENT, "cieg_matrix_upload_shard: null argument");
    if (csb->precision != 0 && csb->precision != 1) cieg::fail(CIEG_ERR_FORMAT, "bad precision tag");
    if (row_lo >= row_hi || row_hi > csb->dim) cieg::fail(CIEG_ERR_DIMENSION, "shard rows outside [0, dim)");
    CIEG_CUDA(cudaSetDevice(ctx->device));
    const std::uint32_t te = choose_tile_edge(csb, group_bounds, ngroups, tile_edge);
    std::vector<std::uint32_t> panels = cieg::plan_panels(csb->dim, group_bounds, ngroups, te);
    cieg::HostTiles ht;
    cieg::build_tiles(*csb, panels, te, ht);
    cieg::restrict_to_rows(ht, row_lo, row_hi);
    *out = upload_tiles(ctx, ht);
    if (group_bounds && ngroups) (*out)->group_bounds_host.assign(group_bounds, group_bounds + ngroups + 1);
  });
}

int cieg_matrix_rows(const cieg_mat* m, uint32_t* row_lo, uint32_t* row_hi, uint32_t* halo_lo, uint32_t* halo_hi) {
  return cieg::guarded([&] {
    if (!m) cieg::fail(CIEG_ERR_ARGUMENT, "null matrix");
    if (row_lo) *row_lo = m->row_lo;
    if (row_hi) *row_hi = m->row_hi;
    if (halo_lo) *halo_lo = m->halo_lo;
    if (halo_hi) *halo_hi = m->halo_hi;
  });
}

int cieg_matrix_partial_rows(const cieg_mat* m, uint32_t* lo, uint32_t* hi) {
  return cieg::guarded([&] {
    if (!m) cieg::fail(CIEG_ERR_ARGUMENT, "null matrix");
    if (lo) *lo = m->sp_sched ? m->sp_partial_lo : m->row_lo;
    if (hi) *hi = m->row_lo;
  });
}

int cieg_spmm_partial(cieg_ctx* ctx, const cieg_mat* mat, const double* x_dev, double* y_dev, uint32_t m,
                      double* yhalo_dev) {
  return cieg::guarded([&] {
    if (!ctx || !mat) cieg::fail(CIEG_ERR_ARGUMENT, "cieg_spmm_partial: null handle");
    if ((!x_dev || !y_dev) && m > 0 && mat->dim > 0) cieg::fail(CIEG_ERR_ARGUMENT, "cieg_spmm_partial: null vector");
    if (x_dev == y_dev && m > 0) cieg::fail(CIEG_ERR_ARGUMENT, "cieg_spmm_partial: X and U must not alias");
    if (!mat->sp_sched) cieg::fail(CIEG_ERR_CONFIG, "cieg_spmm_partial: matrix has no single-pass schedule");
    const bool shard = mat->row_lo != 0 || mat->row_hi != mat->dim;
    if (shard) {
      if (!yhalo_dev && mat->row_lo > mat->sp_partial_lo && m > 0)
        cieg::fail(CIEG_ERR_ARGUMENT, "cieg_spmm_partial: null partial buffer");
      cieg::launch_spmm(ctx, mat, x_dev, m, y_dev, m, m, yhalo_dev, m, true);
    } else {
      const int saved = ctx->spmm_mode;
      ctx->spmm_mode = CIEG_SPMM_SINGLE_PASS;
      try {
        cieg::launch_spmm(ctx, mat, x_dev, m, y_dev, m, m);
      } catch (...) {
        ctx->spmm_mode = saved;
        throw;
      }
      ctx->spmm_mode = saved;
    }
  });
}

int cieg_shard_plan(const cieg_csb_view* csb, const uint32_t* group_bounds, uint32_t ngroups, uint32_t tile_edge,
                    uint32_t nranks, uint32_t* row_bounds, uint32_t* halo_lo, uint32_t* halo_hi) {
  return cieg::guarded([&] {
    if (!csb || !row_bounds || !halo_lo || !halo_hi) cieg::fail(CIEG_ERR_ARGUMENT, "cieg_shard_plan: null argument");
    const std::uint32_t te = choose_tile_edge(csb, group_bounds, ngroups, tile_edge);
    cieg::shard_plan(*csb, group_bounds, ngroups, te, nranks, row_bounds, halo_lo, halo_hi);
  });
}

int cieg_ctx_set_exact_order(cieg_ctx* ctx, int exact) {
  return cieg::guarded([&] {
    if (!ctx) cieg::fail(CIEG_ERR_ARGUMENT, "null context");
    ctx->exact_order = exact ? 1 : 0;
  });
}

int cieg_ctx_set_spmm_mode(cieg_ctx* ctx, int mode) {
  return cieg::guarded([&] {
    if (!ctx) cieg::fail(CIEG_ERR_ARGUMENT, "null context");
    if (mode < CIEG_SPMM_AUTO || mode > CIEG_SPMM_SLICED) cieg::fail(CIEG_ERR_ARGUMENT, "unknown SpMM mode");
    ctx->spmm_mode = mode;
  });
}

int cieg_spmm_effective_mode(cieg_ctx* ctx, cieg_mat* mat, uint32_t m, int* mode) {
  return cieg::guarded([&] {
    if (!ctx || !mat || !mode) cieg::fail(CIEG_ERR_ARGUMENT, "cieg_spmm_effective_mode: null argument");
    *mode = cieg::spmm_effective_mode(ctx, mat, std::min<std::uint32_t>(std::max<std::uint32_t>(m, 1), 16));
  });
}

int cieg_ctx_set_stream(cieg_ctx* ctx, void* stream) {
  return cieg::guarded([&] {
    if (!ctx) cieg::fail(CIEG_ERR_ARGUMENT, "null context");
    CIEG_CUDA(cudaStreamSynchronize(ctx->stream));
    ctx->stream = stream ? static_cast<cudaStream_t>(stream) : ctx->own_stream;
  });
}

int cieg_matrix_destroy(cieg_mat* mat) {
  if (mat) {
    cudaSetDevice(mat->ctx->device);
    cudaStreamSynchronize(mat->ctx->stream);
    delete mat;
  }
  return CIEG_OK;
}

int cieg_matrix_info(const cieg_mat* m, uint32_t* dim, uint64_t* nnz, uint32_t* npanels,
                     uint64_t* ntiles, uint32_t* tile_edge, int* precision, uint64_t* bytes) {
  return cieg::guarded([&] {
    if (!m) cieg::fail(CIEG_ERR_ARGUMENT, "null matrix");
    if (dim) *dim = m->dim;
    if (nnz) *nnz = m->nnz;
    if (npanels) *npanels = m->npanels;
    if (ntiles) *ntiles = m->ntiles;
    if (tile_edge) *tile_edge = m->tile_edge;
    if (precision) *precision = m->precision;
    if (bytes) *bytes = m->tile_bytes;
  });
}

int cieg_spmm(cieg_ctx* ctx, const cieg_mat* mat, const double* x_dev, double* y_dev, uint32_t m) {
  return cieg::guarded([&] {
    if (!ctx || !mat) cieg::fail(CIEG_ERR_ARGUMENT, "cieg_spmm: null handle");
    if ((!x_dev || !y_dev) && m > 0 && mat->dim > 0) cieg::fail(CIEG_ERR_ARGUMENT, "cieg_spmm: null vector");
    if (x_dev == y_dev && m > 0) cieg::fail(CIEG_ERR_ARGUMENT, "cieg_spmm: X and U must not alias");
    cieg::launch_spmm(ctx, mat, x_dev, m, y_dev, m, m);
  });
}


namespace {

bool host_pinned(const void* p) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost || a.type == cudaMemoryTypeManaged;
}

// Host copy of one staging chunk, split over the OpenMP threads.
void par_copy(void* dst, const void* src, std::size_t bytes) {
  constexpr std::size_t kPiece = 256u << 10;  // (an 8 MB staging chunk keeps every thread busy)
  const std::int64_t pieces = static_cast<std::int64_t>((bytes + kPiece - 1) / kPiece);
#pragma omp parallel for schedule(static) if (pieces > 1)
  for (std::int64_t i = 0; i < pieces; ++i) {
    const std::size_t o = static_cast<std::size_t>(i) * kPiece;
    std::memcpy(static_cast<char*>(dst) + o, static_cast<const char*>(src) + o, std::min(kPiece, bytes - o));
  }
}

// The same with non-temporal stores: the copy out of the pinned ring into the
// caller's U (hundreds of MB, not read again soon) skips the read-for-ownership
// of the destination lines and leaves the cache to the staging rings.
void stream_piece(char* dst, const char* src, std::size_t bytes) {
#if defined(__SSE2__)
  const std::size_t head = std::min(bytes, (16 - (reinterpret_cast<std::uintptr_t>(dst) & 15)) & 15);
  std::memcpy(dst, src, head);
  dst += head, src += head, bytes -= head;
  const std::size_t body = bytes & ~static_cast<std::size_t>(63);
  for (std::size_t o = 0; o < body; o += 64) {
    const __m128i a = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + o));
    const __m128i b = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + o + 16));
    const __m128i c = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + o + 32));
    const __m128i d = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + o + 48));
    _mm_stream_si128(reinterpret_cast<__m128i*>(dst + o), a);
    _mm_stream_si128(reinterpret_cast<__m128i*>(dst + o + 16), b);
    _mm_stream_si128(reinterpret_cast<__m128i*>(dst + o + 32), c);
    _mm_stream_si128(reinterpret_cast<__m128i*>(dst + o + 48), d);
  }
  _mm_sfence();
  std::memcpy(dst + body, src + body, bytes - body);
#else
  std::memcpy(dst, src, bytes);
#endif
}

void par_copy_stream(void* dst, const void* src, std::size_t bytes) {
  constexpr std::size_t kPiece = 256u << 10;
  const std::int64_t pieces = static_cast<std::int64_t>((bytes + kPiece - 1) / kPiece);
#pragma omp parallel for schedule(static) if (pieces > 1)
  for (std::int64_t i = 0; i < pieces; ++i) {
    const std::size_t o = static_cast<std::size_t>(i) * kPiece;
    stream_piece(static_cast<char*>(dst) + o, static_cast<const char*>(src) + o, std::min(kPiece, bytes - o));
  }
}

constexpr int kStageSlots = 4;
constexpr std::size_t kStageChunk = 8u << 20;

char* stage_ring(cieg_ctx* ctx) {
  for (auto& e : ctx->stage_ev)
    if (!e) CIEG_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  return static_cast<char*>(ctx->pinned_stage.get(kStageSlots * kStageChunk));
}

// Pageable host -> device through the pinned ring: the host copy of chunk c+1
// (all threads) overlaps the DMA of chunk c.
void upload_staged(cieg_ctx* ctx, void* dst, const void* src, std::size_t bytes) {
  char* ring = stage_ring(ctx);
  const std::size_t chunks = (bytes + kStageChunk - 1) / kStageChunk;
  for (std::size_t c = 0; c < chunks; ++c) {
    const int slot = static_cast<int>(c % kStageSlots);
    const std::size_t off = c * kStageChunk, len = std::min(kStageChunk, bytes - off);
    if (c >= kStageSlots) CIEG_CUDA(cudaEventSynchronize(ctx->stage_ev[slot]));
    par_copy(ring + slot * kStageChunk, static_cast<const char*>(src) + off, len);
    CIEG_CUDA(cudaMemcpyAsync(static_cast<char*>(dst) + off, ring + slot * kStageChunk, len, cudaMemcpyHostToDevice,
                              ctx->stream));
    CIEG_CUDA(cudaEventRecord(ctx->stage_ev[slot], ctx->stream));
  }
}

// Device -> pageable host: kStageSlots chunk DMAs in flight ahead of the host
// copies out of the ring.
void download_staged(cieg_ctx* ctx, void* dst, const void* src, std::size_t bytes) {
  char* ring = stage_ring(ctx);
  const std::size_t chunks = (bytes + kStageChunk - 1) / kStageChunk;
  auto issue = [&](std::size_t c) {
    const int slot = static_cast<int>(c % kStageSlots);
    const std::size_t off = c * kStageChunk, len = std::min(kStageChunk, bytes - off);
    CIEG_CUDA(cudaMemcpyAsync(ring + slot * kStageChunk, static_cast<const char*>(src) + off, len,
                              cudaMemcpyDeviceToHost, ctx->stream));
    CIEG_CUDA(cudaEventRecord(ctx->stage_ev[slot], ctx->stream));
  };
  for (std::size_t c = 0; c < chunks && c < kStageSlots; ++c) issue(c);
  for (std::size_t c = 0; c < chunks; ++c) {
    const int slot = static_cast<int>(c % kStageSlots);
    const std::size_t off = c * kStageChunk, len = std::min(kStageChunk, bytes - off);
    CIEG_CUDA(cudaEventSynchronize(ctx->stage_ev[slot]));
    par_copy_stream(static_cast<char*>(dst) + off, ring + slot * kStageChunk, len);
    if (c + kStageSlots < chunks) issue(c + kStageSlots);
  }
}

}  // namespace

}  // extern "C"

namespace cieg {

// ---- pageable host buffers of the pipelined host SpMM (context.hpp)
namespace {
void copy_pieces(void* dst, const void* src, std::size_t bytes, int threads, bool stream) {
  constexpr std::size_t kPiece = 256u << 10;
  const std::int64_t pieces = static_cast<std::int64_t>((bytes + kPiece - 1) / kPiece);
#pragma omp parallel for schedule(static) num_threads(threads) if (pieces > 1)
  for (std::int64_t i = 0; i < pieces; ++i) {
    const std::size_t o = static_cast<std::size_t>(i) * kPiece, len = std::min(kPiece, bytes - o);
    if (stream)
      stream_piece(static_cast<char*>(dst) + o, static_cast<const char*>(src) + o, len);
    else
      std::memcpy(static_cast<char*>(dst) + o, static_cast<const char*>(src) + o, len);
  }
}
}  // namespace

struct HostCopier {
  struct Job {
    cudaEvent_t ev;
    char* dst;
    const char* src;
    std::size_t len;
  };
  std::thread th;
  std::mutex mu;
  std::condition_variable cv_job, cv_done;
  std::deque<Job> q;
  std::size_t submitted = 0, retired = 0;
  bool stop = false;
  std::string error;
  int device = 0, threads = 1;
  void run() {
    cudaSetDevice(device);
    for (;;) {
      Job j;
      {
        std::unique_lock<std::mutex> lk(mu);
        cv_job.wait(lk, [&] { return stop || !q.empty(); });
        if (q.empty()) return;
        j = q.front();
        q.pop_front();
      }
      const cudaError_t e = cudaEventSynchronize(j.ev);
      if (e == cudaSuccess) copy_pieces(j.dst, j.src, j.len, threads, true);
      {
        std::lock_guard<std::mutex> lk(mu);
        if (e != cudaSuccess && error.empty()) error = cudaGetErrorString(e);
        ++retired;
      }
      cv_done.notify_all();
    }
  }
};

namespace {
// OpenMP threads of the helper's copy-out; the rest copy X into the upload
// ring (CIEG_COPIER_THREADS overrides). Measured on config 2, m = 16, 16
// cores, both buffers pageable: 2 / 4 / 6 / 8 helper threads = 18.9 / 15.6 /
// 12.1 / 11.3 ms per call -- with both DMA directions running, either copy
// needs half the cores (alone, four threads stream 74 GB/s).
int copier_threads() {
  static const int n = [] {
    const int all = std::max(1, omp_get_max_threads());
    if (const char* e = std::getenv("CIEG_COPIER_THREADS")) return std::max(1, std::min(all, std::atoi(e)));
    return std::max(1, all / 2);
  }();
  return n;
}
HostCopier* copier(cieg_ctx* ctx) {
  if (!ctx->copier) {
    auto* c = new HostCopier;
    c->device = ctx->device;
    c->threads = copier_threads();
    c->th = std::thread([c] { c->run(); });
    ctx->copier = c;
  }
  return ctx->copier;
}
}  // namespace

void host_copy_in(void* dst, const void* src, std::size_t bytes, bool shared) {
  const int all = std::max(1, omp_get_max_threads());
  copy_pieces(dst, src, bytes, shared ? std::max(1, all - copier_threads()) : all, false);
}

std::size_t copier_submit(cieg_ctx* ctx, cudaEvent_t ev, void* dst, const void* src, std::size_t bytes) {
  HostCopier* c = copier(ctx);
  std::size_t n;
  {
    std::lock_guard<std::mutex> lk(c->mu);
    c->q.push_back(HostCopier::Job{ev, static_cast<char*>(dst), static_cast<const char*>(src), bytes});
    n = ++c->submitted;
  }
  c->cv_job.notify_one();
  return n;
}

std::size_t copier_submitted(cieg_ctx* ctx) {
  HostCopier* c = copier(ctx);
  std::lock_guard<std::mutex> lk(c->mu);
  return c->submitted;
}

void copier_wait(cieg_ctx* ctx, std::size_t jobs) {
  HostCopier* c = copier(ctx);
  std::unique_lock<std::mutex> lk(c->mu);
  c->cv_done.wait(lk, [&] { return c->retired >= jobs; });
  if (!c->error.empty()) {
    const std::string msg = "download copy: " + c->error;
    c->error.clear();
    lk.unlock();
    fail(CIEG_ERR_CUDA, msg);
  }
}

void copier_drain(cieg_ctx* ctx) noexcept {
  if (!ctx->copier) return;
  HostCopier* c = ctx->copier;
  std::unique_lock<std::mutex> lk(c->mu);
  c->cv_done.wait(lk, [&] { return c->retired >= c->submitted; });
  c->error.clear();
}

void destroy_copier(cieg_ctx* ctx) {
  if (!ctx->copier) return;
  HostCopier* c = ctx->copier;
  {
    std::lock_guard<std::mutex> lk(c->mu);
    c->stop = true;
  }
  c->cv_job.notify_all();
  if (c->th.joinable()) c->th.join();
  delete c;
  ctx->copier = nullptr;
}

}  // namespace cieg

extern "C" {

// ci::spmm's host call (the drop-in binds it, integration/ci_gpu_dropin.cpp):
// pinned host buffers go straight to the copy engines; pageable ones (the
// std::vector inside ci::BlockVectors) stream through a pinned chunk ring
// with the host copies spread over the OpenMP threads.
int cieg_spmm_host(cieg_ctx* ctx, const cieg_mat* mat, const double* x_host, double* y_host,
                   uint32_t m) {
  return cieg::guarded([&] {
    if (!ctx || !mat) cieg::fail(CIEG_ERR_ARGUMENT, "cieg_spmm_host: null handle");
    const std::size_t xbytes = static_cast<std::size_t>(mat->dim) * m * sizeof(double);
    const std::size_t ybytes = static_cast<std::size_t>(mat->row_hi - mat->row_lo) * m * sizeof(double);
    if (xbytes == 0) return;
    if (!x_host || !y_host) cieg::fail(CIEG_ERR_ARGUMENT, "cieg_spmm_host: null vector");
    CIEG_CUDA(cudaSetDevice(ctx->device));
    const bool x_pinned = host_pinned(x_host), y_pinned = host_pinned(y_host);
    // the sliced kernel: upload, kernels and download pipelined over row chunks
    if (m <= 16 && cieg::sliced_spmm_host(ctx, const_cast<cieg_mat*>(mat), x_host, y_host, m, x_pinned, y_pinned))
      return;
    double* dx = static_cast<double*>(ctx->scratch_x.get(xbytes));
    double* dy = static_cast<double*>(ctx->scratch_y.get(ybytes));
    if (x_pinned)
      CIEG_CUDA(cudaMemcpyAsync(dx, x_host, xbytes, cudaMemcpyHostToDevice, ctx->stream));
    else
      upload_staged(ctx, dx, x_host, xbytes);
    cieg::launch_spmm(ctx, mat, dx, m, dy, m, m);
    if (y_pinned)
      CIEG_CUDA(cudaMemcpyAsync(y_host, dy, ybytes, cudaMemcpyDeviceToHost, ctx->stream));
    else
      download_staged(ctx, y_host, dy, ybytes);
    CIEG_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

int cieg_spmm_host_batch(cieg_ctx* ctx, const cieg_mat* mat, const double* const* x_hosts, double* const* y_hosts,
                         uint32_t m, uint32_t count) {
  return cieg::guarded([&] {
    if (!ctx || !mat || (count && (!x_hosts || !y_hosts)))
      cieg::fail(CIEG_ERR_ARGUMENT, "cieg_spmm_host_batch: null argument");
    const std::size_t xbytes = static_cast<std::size_t>(mat->dim) * m * sizeof(double);
    const std::size_t ybytes = static_cast<std::size_t>(mat->row_hi - mat->row_lo) * m * sizeof(double);
    if (xbytes == 0 || count == 0) return;
    for (uint32_t i = 0; i < count; ++i)
      if (!x_hosts[i] || !y_hosts[i]) cieg::fail(CIEG_ERR_ARGUMENT, "cieg_spmm_host_batch: null vector");
    CIEG_CUDA(cudaSetDevice(ctx->device));
    // Three device X / U buffers: the upload of X_{i+1}, K1 on U_i and the
    // download of U_{i-1} run concurrently without waiting on each other's
    // buffer reuse (the download of a U takes longer than K1 when both copy
    // directions are busy).
    constexpr int kB = 3;
    double* dx[kB] = {static_cast<double*>(ctx->scratch_x.get(xbytes)), static_cast<double*>(ctx->scratch_x2.get(xbytes)),
                      static_cast<double*>(ctx->scratch_x3.get(xbytes))};
    double* dy[kB] = {static_cast<double*>(ctx->scratch_y.get(ybytes)), static_cast<double*>(ctx->scratch_y2.get(ybytes)),
                      static_cast<double*>(ctx->scratch_y3.get(ybytes))};
    cudaStream_t up = nullptr, down = nullptr;
    cudaEvent_t uploaded[kB] = {}, computed[kB] = {}, downloaded[kB] = {};
    auto cleanup = [&] {
      for (int b = 0; b < kB; ++b) {
        if (uploaded[b]) cudaEventDestroy(uploaded[b]);
        if (computed[b]) cudaEventDestroy(computed[b]);
        if (downloaded[b]) cudaEventDestroy(downloaded[b]);
      }
      if (up) cudaStreamDestroy(up);
      if (down) cudaStreamDestroy(down);
    };
    try {
      CIEG_CUDA(cudaStreamCreateWithFlags(&up, cudaStreamNonBlocking));
      CIEG_CUDA(cudaStreamCreateWithFlags(&down, cudaStreamNonBlocking));
      for (int b = 0; b < kB; ++b) {
        CIEG_CUDA(cudaEventCreateWithFlags(&uploaded[b], cudaEventDisableTiming));
        CIEG_CUDA(cudaEventCreateWithFlags(&computed[b], cudaEventDisableTiming));
        CIEG_CUDA(cudaEventCreateWithFlags(&downloaded[b], cudaEventDisableTiming));
        // nothing may touch the buffers before work already queued on the context stream
        CIEG_CUDA(cudaEventRecord(computed[b], ctx->stream));
        CIEG_CUDA(cudaEventRecord(downloaded[b], ctx->stream));
      }
      for (uint32_t i = 0; i < count; ++i) {
        const int b = static_cast<int>(i % kB);
        CIEG_CUDA(cudaStreamWaitEvent(up, computed[b], 0));  // K1 of step i-3 has read X[b]
        CIEG_CUDA(cudaMemcpyAsync(dx[b], x_hosts[i], xbytes, cudaMemcpyHostToDevice, up));
        CIEG_CUDA(cudaEventRecord(uploaded[b], up));
        CIEG_CUDA(cudaStreamWaitEvent(ctx->stream, uploaded[b], 0));
        CIEG_CUDA(cudaStreamWaitEvent(ctx->stream, downloaded[b], 0));  // U[b] of step i-3 is home
        cieg::launch_spmm(ctx, mat, dx[b], m, dy[b], m, m);
        CIEG_CUDA(cudaEventRecord(computed[b], ctx->stream));
        CIEG_CUDA(cudaStreamWaitEvent(down, computed[b], 0));
        CIEG_CUDA(cudaMemcpyAsync(y_hosts[i], dy[b], ybytes, cudaMemcpyDeviceToHost, down));
        CIEG_CUDA(cudaEventRecord(downloaded[b], down));
      }
      CIEG_CUDA(cudaStreamSynchronize(down));
      CIEG_CUDA(cudaStreamSynchronize(ctx->stream));
      CIEG_CUDA(cudaStreamSynchronize(up));
    } catch (...) {
      cleanup();
      throw;
    }
    cleanup();
  });
}

}  // extern "C"
