// nccl_plane.cpp -- the sharded solver's data plane inside the library: the
// collectives of SURVEY.md 8(e) (the reference planner's fused mode,
// proj/src/planner.cpp:116-122) on an NCCL communicator owned by the
// context, on the context's stream, with no host round trip except the Gram
// results the host loop needs anyway:
//   * Gram all-reduce: ncclAllReduce of the <= 48 x 48 device result before
//     its single D2H (cieg::gram / combine_gram, blockvec.cu);
//   * X halo exchange before every SpMM: grouped ncclSend / ncclRecv of
//     exactly the rows each peer's shard reads (its halo minus its own rows);
//   * single-pass partial reduction after it: the transposed partials for
//     lower ranks' rows travel to their owners, grouped send / recv, added in
//     ascending rank order (deterministic for a fixed partition).
// libnccl is opened at run time (dlopen "libnccl.so.2"): the library has no
// link-time NCCL dependency, and inside a torch process it binds to the
// libnccl torch already loaded (same soname).
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

#include "context.hpp"

namespace cieg {

struct NcclPlane {
  void* lib = nullptr;
  ncclComm_t comm = nullptr;
  int rank = 0, nranks = 1;
  decltype(&ncclGetUniqueId) get_unique_id = nullptr;
  decltype(&ncclCommInitRank) init_rank = nullptr;
  decltype(&ncclCommDestroy) destroy = nullptr;
  decltype(&ncclAllReduce) all_reduce = nullptr;
  decltype(&ncclAllGather) all_gather = nullptr;
  decltype(&ncclSend) send = nullptr;
  decltype(&ncclRecv) recv = nullptr;
  decltype(&ncclGroupStart) group_start = nullptr;
  decltype(&ncclGroupEnd) group_end = nullptr;
  decltype(&ncclGetErrorString) error_string = nullptr;
  DevBuf scratch;
};

namespace {

NcclPlane* open_nccl() {
  auto* p = new NcclPlane;
  p->lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!p->lib) {
    delete p;
    fail(CIEG_ERR_CONFIG, std::string("NCCL unavailable: ") + dlerror());
  }
  auto sym = [&](const char* name) {
    void* f = dlsym(p->lib, name);
    if (!f) fail(CIEG_ERR_CONFIG, std::string("NCCL symbol missing: ") + name);
    return f;
  };
  p->get_unique_id = reinterpret_cast<decltype(&ncclGetUniqueId)>(sym("ncclGetUniqueId"));
  p->init_rank = reinterpret_cast<decltype(&ncclCommInitRank)>(sym("ncclCommInitRank"));
  p->destroy = reinterpret_cast<decltype(&ncclCommDestroy)>(sym("ncclCommDestroy"));
  p->all_reduce = reinterpret_cast<decltype(&ncclAllReduce)>(sym("ncclAllReduce"));
  p->all_gather = reinterpret_cast<decltype(&ncclAllGather)>(sym("ncclAllGather"));
  p->send = reinterpret_cast<decltype(&ncclSend)>(sym("ncclSend"));
  p->recv = reinterpret_cast<decltype(&ncclRecv)>(sym("ncclRecv"));
  p->group_start = reinterpret_cast<decltype(&ncclGroupStart)>(sym("ncclGroupStart"));
  p->group_end = reinterpret_cast<decltype(&ncclGroupEnd)>(sym("ncclGroupEnd"));
  p->error_string = reinterpret_cast<decltype(&ncclGetErrorString)>(sym("ncclGetErrorString"));
  return p;
}

void check(const NcclPlane* p, ncclResult_t r, const char* what) {
  if (r != ncclSuccess) fail(CIEG_ERR_CUDA, std::string(what) + ": " + p->error_string(r));
}

__attribute__((unused)) NcclPlane* plane(cieg_ctx* ctx) {
  if (!ctx->nccl) fail(CIEG_ERR_CONFIG, "no NCCL communicator on this context (cieg_ctx_nccl_init)");
  return ctx->nccl;
}

// Row ranges of every rank's shard: owned [lo, hi), read [halo_lo, halo_hi),
// single-pass partial rows [part_lo, lo).
struct Ranges {
  std::uint32_t lo, hi, halo_lo, halo_hi, part_lo, pad[3];
};

}  // namespace

bool nccl_active(const cieg_ctx* ctx) { return ctx->nccl != nullptr && ctx->nccl_grams; }

void nccl_allreduce_sum(cieg_ctx* ctx, double* dev, std::size_t count) {
  NcclPlane* p = plane(ctx);
  if (count == 0) return;
  check(p, p->all_reduce(dev, dev, count, ncclDouble, ncclSum, p->comm, ctx->stream), "ncclAllReduce");
}

void destroy_nccl(cieg_ctx* ctx) {
  if (!ctx->nccl) return;
  if (ctx->nccl->comm) ctx->nccl->destroy(ctx->nccl->comm);
  ctx->nccl->scratch.release();
  delete ctx->nccl;
  ctx->nccl = nullptr;
}

namespace {

std::vector<Ranges> gather_ranges(cieg_ctx* ctx, const cieg_mat* m) {
  NcclPlane* p = plane(ctx);
  Ranges mine{m->row_lo, m->row_hi, m->halo_lo, m->halo_hi, m->sp_partial_lo, {0, 0, 0}};
  auto* d = static_cast<Ranges*>(p->scratch.get(sizeof(Ranges) * (p->nranks + 1)));
  CIEG_CUDA(cudaMemcpyAsync(d + p->nranks, &mine, sizeof(Ranges), cudaMemcpyHostToDevice, ctx->stream));
  check(p, p->all_gather(d + p->nranks, d, sizeof(Ranges) / sizeof(std::uint32_t), ncclUint32, p->comm, ctx->stream),
        "ncclAllGather");
  std::vector<Ranges> all(p->nranks);
  CIEG_CUDA(cudaMemcpyAsync(all.data(), d, sizeof(Ranges) * p->nranks, cudaMemcpyDeviceToHost, ctx->stream));
  CIEG_CUDA(cudaStreamSynchronize(ctx->stream));
  return all;
}

__global__ void add_rows_kernel(double* y, const double* r, std::uint64_t count) {
  for (std::uint64_t e = blockIdx.x * std::uint64_t(blockDim.x) + threadIdx.x; e < count;
       e += std::uint64_t(gridDim.x) * blockDim.x)
    y[e] += r[e];
}

}  // namespace

// The native hooks of a sharded solve (cieg_dist_hooks signatures).
struct NcclSolve {
  cieg_ctx* ctx;
  const cieg_mat* mat;
  std::vector<Ranges> ranges;
  DevBuf recv;
};

int nccl_hook_allreduce(void* user, double* host_buf, std::uint64_t count) {
  auto* s = static_cast<NcclSolve*>(user);
  return guarded([&] {
    NcclPlane* p = plane(s->ctx);
    auto* d = static_cast<double*>(p->scratch.get(sizeof(double) * std::max<std::uint64_t>(1, count)));
    CIEG_CUDA(cudaMemcpyAsync(d, host_buf, sizeof(double) * count, cudaMemcpyHostToDevice, s->ctx->stream));
    nccl_allreduce_sum(s->ctx, d, count);
    CIEG_CUDA(cudaMemcpyAsync(host_buf, d, sizeof(double) * count, cudaMemcpyDeviceToHost, s->ctx->stream));
    CIEG_CUDA(cudaStreamSynchronize(s->ctx->stream));
  });
}

int nccl_hook_gather(void* user, const double* x_local, std::uint32_t m, double* full) {
  auto* s = static_cast<NcclSolve*>(user);
  return guarded([&] {
    NcclPlane* p = plane(s->ctx);
    const Ranges& me = s->ranges[p->rank];
    const std::size_t own = static_cast<std::size_t>(me.hi - me.lo) * m;
    if (own)
      CIEG_CUDA(cudaMemcpyAsync(full + static_cast<std::size_t>(me.lo) * m, x_local, sizeof(double) * own,
                                cudaMemcpyDeviceToDevice, s->ctx->stream));
    check(p, p->group_start(), "ncclGroupStart");
    for (int q = 0; q < p->nranks; ++q) {
      if (q == p->rank) continue;
      const Ranges& o = s->ranges[q];
      const std::uint32_t sa = std::max(me.lo, o.halo_lo), sb = std::min(me.hi, o.halo_hi);
      if (sa < sb)
        check(p, p->send(x_local + static_cast<std::size_t>(sa - me.lo) * m, static_cast<std::size_t>(sb - sa) * m,
                         ncclDouble, q, p->comm, s->ctx->stream),
              "ncclSend");
      const std::uint32_t ra = std::max(o.lo, me.halo_lo), rb = std::min(o.hi, me.halo_hi);
      if (ra < rb)
        check(p, p->recv(full + static_cast<std::size_t>(ra) * m, static_cast<std::size_t>(rb - ra) * m, ncclDouble, q,
                         p->comm, s->ctx->stream),
              "ncclRecv");
    }
    check(p, p->group_end(), "ncclGroupEnd");
  });
}

int nccl_hook_reduce_partials(void* user, const double* yhalo, std::uint32_t m, double* y_local) {
  auto* s = static_cast<NcclSolve*>(user);
  return guarded([&] {
    NcclPlane* p = plane(s->ctx);
    const Ranges& me = s->ranges[p->rank];
    // receive slots: the partials higher ranks computed for this rank's rows
    std::vector<std::size_t> off(p->nranks + 1, 0);
    for (int q = 0; q < p->nranks; ++q) {
      const Ranges& o = s->ranges[q];
      const std::uint32_t a = std::max(o.part_lo, me.lo), b = std::min(o.lo, me.hi);
      off[q + 1] = off[q] + (q > p->rank && a < b ? static_cast<std::size_t>(b - a) * m : 0);
    }
    auto* rbuf = static_cast<double*>(s->recv.get(sizeof(double) * std::max<std::size_t>(1, off[p->nranks])));
    check(p, p->group_start(), "ncclGroupStart");
    for (int q = 0; q < p->nranks; ++q) {
      if (q == p->rank) continue;
      const Ranges& o = s->ranges[q];
      if (q < p->rank) {  // this rank's partials for q's rows
        const std::uint32_t a = std::max(me.part_lo, o.lo), b = std::min(me.lo, o.hi);
        if (a < b)
          check(p, p->send(yhalo + static_cast<std::size_t>(a - me.part_lo) * m, static_cast<std::size_t>(b - a) * m,
                           ncclDouble, q, p->comm, s->ctx->stream),
                "ncclSend");
      } else if (off[q + 1] > off[q]) {
        check(p, p->recv(rbuf + off[q], off[q + 1] - off[q], ncclDouble, q, p->comm, s->ctx->stream), "ncclRecv");
      }
    }
    check(p, p->group_end(), "ncclGroupEnd");
    for (int q = p->rank + 1; q < p->nranks; ++q) {  // ascending rank order
      if (off[q + 1] == off[q]) continue;
      const Ranges& o = s->ranges[q];
      const std::uint32_t a = std::max(o.part_lo, me.lo);
      const std::uint64_t count = off[q + 1] - off[q];
      add_rows_kernel<<<static_cast<unsigned>(std::min<std::uint64_t>((count + 255) / 256, 4ull * s->ctx->sm_count)),
                        256, 0, s->ctx->stream>>>(y_local + static_cast<std::size_t>(a - me.lo) * m, rbuf + off[q],
                                                  count);
      CIEG_CUDA(cudaGetLastError());
      ++s->ctx->launches;
    }
  });
}

NcclSolve* nccl_solve_begin(cieg_ctx* ctx, const cieg_mat* mat) {
  plane(ctx);
  auto* s = new NcclSolve{ctx, mat, {}, {}};
  try {
    s->ranges = gather_ranges(ctx, mat);
  } catch (...) {
    delete s;
    throw;
  }
  ctx->nccl_grams = true;
  return s;
}

void nccl_solve_end(NcclSolve* s) {
  if (!s) return;
  s->ctx->nccl_grams = false;
  s->recv.release();
  delete s;
}

}  // namespace cieg

extern "C" {

int cieg_nccl_unique_id(uint8_t* id_out) {
  return cieg::guarded([&] {
    if (!id_out) cieg::fail(CIEG_ERR_ARGUMENT, "cieg_nccl_unique_id: null buffer");
    cieg::NcclPlane* p = cieg::open_nccl();
    ncclUniqueId id;
    const ncclResult_t r = p->get_unique_id(&id);
    std::string err = r == ncclSuccess ? "" : p->error_string(r);
    delete p;
    if (!err.empty()) cieg::fail(CIEG_ERR_CUDA, "ncclGetUniqueId: " + err);
    std::memcpy(id_out, &id, sizeof(id));
  });
}

int cieg_ctx_nccl_init(cieg_ctx* ctx, const uint8_t* id, int nranks, int rank) {
  return cieg::guarded([&] {
    if (!ctx || !id) cieg::fail(CIEG_ERR_ARGUMENT, "cieg_ctx_nccl_init: null argument");
    if (nranks < 1 || rank < 0 || rank >= nranks) cieg::fail(CIEG_ERR_ARGUMENT, "cieg_ctx_nccl_init: bad rank");
    cieg::destroy_nccl(ctx);
    CIEG_CUDA(cudaSetDevice(ctx->device));
    cieg::NcclPlane* p = cieg::open_nccl();
    ncclUniqueId uid;
    std::memcpy(&uid, id, sizeof(uid));
    const ncclResult_t r = p->init_rank(&p->comm, nranks, uid, rank);
    if (r != ncclSuccess) {
      std::string err = p->error_string(r);
      delete p;
      cieg::fail(CIEG_ERR_CUDA, "ncclCommInitRank: " + err);
    }
    p->rank = rank;
    p->nranks = nranks;
    ctx->nccl = p;
  });
}

int cieg_ctx_nccl_finalize(cieg_ctx* ctx) {
  return cieg::guarded([&] {
    if (!ctx) cieg::fail(CIEG_ERR_ARGUMENT, "null context");
    cieg::destroy_nccl(ctx);
  });
}

}  // extern "C"
