// Row-band sharding of optimize_level over GPUs,
// orchestrated in the library with NCCL on the context stream.
//
// The reference has no spatial parallelism (its only parallelism is the
// search_step thread fan-out, optimizer.cpp:314-330).  Here the output rows
// are split into contiguous bands aligned to anchor rows (psg_shard_plan); the
// exemplar, PCA model and tree are replicated; one EM iteration is the band's
// four phases (runtime.cpp) with three exchanges, all enqueued on the context
// stream so they are ordered against the kernels that fill and read their
// buffers:
//   1. histogram bin counts: ncclAllReduce(sum) of u64 (exact integers);
//   2. (eff, idx) of the anchor rows the next band's pixels need: ncclSend to
//      rank + 1 / ncclRecv from rank - 1 (the M-step then accumulates every
//      covering anchor in ascending id: bit-identical to one device);
//   3. the first fp32 mirror rows: ncclSend to rank - 1 / ncclRecv from
//      rank + 1 (the halo rows the band's windows read);
//   4. the nine telemetry partials: ncclAllGather, summed in rank order (so
//      every rank takes the same convergence decision from the exact global
//      `changed` and reports identical statistics).
// NCCL is loaded at communicator creation (dlopen "libnccl.so.2": the one
// torch already loaded in-process, or the system's), so the library carries no
// link-time NCCL dependency.  A loopback variant runs `world` bands of one
// image in this process with device copies for the exchanges: the same
// schedule, used to test the exchange buffers on a single GPU.
#include <dlfcn.h>
#include <nccl.h>

#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "psg_internal.h"

namespace psg {
namespace {
struct BandIO;
}
}  // namespace psg

struct psg_comm {
  psg_ctx* ctx = nullptr;
  int world = 1, rank = 0;
  ncclComm_t nccl = nullptr;
  // exchange buffers of the band plan last iterated (reused across calls)
  std::shared_ptr<psg::BandIO> io;
};

namespace psg {
namespace {

struct Nccl {
  void* h = nullptr;
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                             cudaStream_t) = nullptr;
  ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                             cudaStream_t) = nullptr;
  ncclResult_t (*send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*group_start)() = nullptr;
  ncclResult_t (*group_end)() = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
};

const Nccl& nccl() {
  static Nccl n;
  static bool tried = false;
  if (!tried) {
    tried = true;
    // an NCCL already in the process (e.g. the one torch ships) wins; else
    // PERSYN_NCCL (a path), else the system's libnccl.so.2
    n.h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!n.h)
      if (const char* p = std::getenv("PERSYN_NCCL")) n.h = dlopen(p, RTLD_NOW);
    if (!n.h) n.h = dlopen("libnccl.so.2", RTLD_NOW);
    if (!n.h) n.h = dlopen("libnccl.so", RTLD_NOW);
    if (n.h) {
      auto sym = [&](const char* s) { return dlsym(n.h, s); };
      n.get_unique_id = reinterpret_cast<decltype(n.get_unique_id)>(sym("ncclGetUniqueId"));
      n.comm_init_rank = reinterpret_cast<decltype(n.comm_init_rank)>(sym("ncclCommInitRank"));
      n.comm_destroy = reinterpret_cast<decltype(n.comm_destroy)>(sym("ncclCommDestroy"));
      n.all_reduce = reinterpret_cast<decltype(n.all_reduce)>(sym("ncclAllReduce"));
      n.all_gather = reinterpret_cast<decltype(n.all_gather)>(sym("ncclAllGather"));
      n.send = reinterpret_cast<decltype(n.send)>(sym("ncclSend"));
      n.recv = reinterpret_cast<decltype(n.recv)>(sym("ncclRecv"));
      n.group_start = reinterpret_cast<decltype(n.group_start)>(sym("ncclGroupStart"));
      n.group_end = reinterpret_cast<decltype(n.group_end)>(sym("ncclGroupEnd"));
      n.error_string = reinterpret_cast<decltype(n.error_string)>(sym("ncclGetErrorString"));
    }
  }
  if (!n.h || !n.get_unique_id || !n.comm_init_rank || !n.send || !n.group_end)
    fail(PSG_E_NCCL, "NCCL (libnccl.so.2) is not available");
  return n;
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess)
    fail(PSG_E_NCCL, std::string(what) + ": " +
                         (nccl().error_string ? nccl().error_string(r) : "NCCL error"));
}

void check(psg_status s) {
  if (s != PSG_OK) fail(s, psg_last_error());
}

// Exchange buffers and sizes of one band (the plan arithmetic of the
// reference-free band schedule).
struct BandIO {
  psg_band plan{}, up{}, down{};  // this band, rank - 1's, rank + 1's
  int C = 0, slots = 0, bins = 0;
  bool hist = false;
  int send_row0 = 0;
  int64_t n_up = 0, n_halo_ae = 0;  // anchors sent up / received from below
  int n_send_rows = 0, n_halo_rows = 0;
  DBuf<unsigned long long> counts, counts_g;
  DBuf<uint8_t> send_ae, recv_ae;
  DBuf<float> send_rows, recv_rows;
  DBuf<double> part, part_all;

  bool matches(const psg_band& b, int C_, const psg_opt_cfg& cfg, bool hist_on) const {
    return std::memcmp(&plan, &b, sizeof(b)) == 0 && C == C_ && hist == hist_on &&
           (!hist || (bins == cfg.histogram_bins &&
                      slots == (cfg.histogram_include_scale ? C_ : 3)));
  }

  void setup(const psg_band& b, int C_, const psg_opt_cfg& cfg, bool hist_on) {
    plan = b;
    C = C_;
    hist = hist_on;
    bins = cfg.histogram_bins;
    slots = cfg.histogram_include_scale ? C : 3;
    const int r = b.rank, w = b.world;
    if (r > 0) check(psg_shard_plan(b.W, b.H, b.w, b.spacing, r - 1, w, &up));
    if (r + 1 < w) check(psg_shard_plan(b.W, b.H, b.w, b.spacing, r + 1, w, &down));
    send_row0 = r + 1 < w ? down.hlo : b.a1;
    n_up = (int64_t)(b.a1 - send_row0) * b.nx;
    n_halo_ae = (int64_t)(b.a0 - b.hlo) * b.nx;
    n_send_rows = r > 0 ? up.e1 - up.p1 : 0;
    n_halo_rows = b.e1 - b.p1;
    if (hist) {
      counts.alloc((size_t)bins * slots);
      counts_g.alloc((size_t)bins * slots);
    }
    send_ae.alloc((size_t)std::max<int64_t>(1, n_up * 12));
    recv_ae.alloc((size_t)std::max<int64_t>(1, n_halo_ae * 12));
    send_rows.alloc((size_t)std::max(1, n_send_rows) * b.W * C);
    recv_rows.alloc((size_t)std::max(1, n_halo_rows) * b.W * C);
    part.alloc(9);
    part_all.alloc((size_t)9 * w);
  }
};

// One EM iteration of this rank's band over NCCL (everything on ctx->stream).
bool nccl_iteration(psg_level* L, psg_comm* cm, BandIO& io, psg_iter_stats* st, bool honor,
                    int64_t total_anchors, const psg_opt_cfg& cfg, int iter) {
  const Nccl& n = nccl();
  cudaStream_t s = cm->ctx->stream;
  const int r = cm->rank, w = cm->world;
  check(psg_band_phase1(L, io.hist ? io.counts.p : nullptr));
  if (io.hist)
    nccl_check(n.all_reduce(io.counts.p, io.counts_g.p, io.counts.n, ncclUint64, ncclSum, cm->nccl, s),
               "ncclAllReduce(counts)");
  check(psg_band_phase2(L, io.hist ? io.counts_g.p : nullptr, io.send_row0, io.send_ae.p));
  nccl_check(n.group_start(), "ncclGroupStart");
  if (r + 1 < w && io.n_up > 0)
    nccl_check(n.send(io.send_ae.p, (size_t)io.n_up * 12, ncclUint8, r + 1, cm->nccl, s), "ncclSend");
  if (r > 0 && io.n_halo_ae > 0)
    nccl_check(n.recv(io.recv_ae.p, (size_t)io.n_halo_ae * 12, ncclUint8, r - 1, cm->nccl, s),
               "ncclRecv");
  nccl_check(n.group_end(), "ncclGroupEnd");
  check(psg_band_phase3(L, io.n_halo_ae > 0 ? io.recv_ae.p : nullptr, io.n_send_rows,
                        io.n_send_rows > 0 ? io.send_rows.p : nullptr));
  const size_t row = (size_t)io.plan.W * io.C;
  nccl_check(n.group_start(), "ncclGroupStart");
  if (r > 0 && io.n_send_rows > 0)
    nccl_check(n.send(io.send_rows.p, io.n_send_rows * row, ncclFloat32, r - 1, cm->nccl, s),
               "ncclSend");
  if (r + 1 < w && io.n_halo_rows > 0)
    nccl_check(n.recv(io.recv_rows.p, io.n_halo_rows * row, ncclFloat32, r + 1, cm->nccl, s),
               "ncclRecv");
  nccl_check(n.group_end(), "ncclGroupEnd");
  double p[9], all[9 * 64];
  check(psg_band_phase4(L, io.n_halo_rows > 0 ? io.recv_rows.p : nullptr, p));
  if (w > 64) fail(PSG_E_DOMAIN, "at most 64 ranks");
  PSG_CUDA(cudaMemcpyAsync(io.part.p, p, sizeof(p), cudaMemcpyHostToDevice, s));
  nccl_check(n.all_gather(io.part.p, io.part_all.p, 9, ncclFloat64, cm->nccl, s),
             "ncclAllGather(partials)");
  PSG_CUDA(cudaMemcpyAsync(all, io.part_all.p, sizeof(double) * 9 * w, cudaMemcpyDeviceToHost, s));
  PSG_CUDA(cudaStreamSynchronize(s));
  double g[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
  for (int k = 0; k < w; ++k)  // rank order: identical sums on every rank
    for (int j = 0; j < 9; ++j) g[j] += all[9 * k + j];
  check(psg_band_commit(L, g, st));
  return honor && iter >= cfg.min_iterations &&
         g[3] < cfg.convergence_fraction * (double)total_anchors;
}

}  // namespace
}  // namespace psg

using psg::fail;

extern "C" psg_status psg_comm_unique_id(void* id) {
  try {
    if (!id) fail(PSG_E_DOMAIN, "null argument");
    ncclUniqueId u;
    psg::nccl_check(psg::nccl().get_unique_id(&u), "ncclGetUniqueId");
    std::memcpy(id, &u, sizeof(u));
    return PSG_OK;
  } catch (const psg::Error& e) {
    psg::set_last_error(e.what());
    return e.code;
  }
}

extern "C" psg_status psg_comm_create(psg_ctx* ctx, const void* id, int world, int rank,
                                      psg_comm** out) {
  try {
    if (!ctx || !id || !out) fail(PSG_E_DOMAIN, "null argument");
    if (world < 1 || rank < 0 || rank >= world) fail(PSG_E_DOMAIN, "bad rank / world size");
    *out = nullptr;
    PSG_CUDA(cudaSetDevice(ctx->device));
    auto c = std::make_unique<psg_comm>();
    c->ctx = ctx;
    c->world = world;
    c->rank = rank;
    ncclUniqueId u;
    std::memcpy(&u, id, sizeof(u));
    psg::nccl_check(psg::nccl().comm_init_rank(&c->nccl, world, u, rank), "ncclCommInitRank");
    *out = c.release();
    return PSG_OK;
  } catch (const psg::Error& e) {
    psg::set_last_error(e.what());
    return e.code;
  }
}

extern "C" void psg_comm_destroy(psg_comm* comm) {
  if (!comm) return;
  {
    psg::StreamScope _ss(comm->ctx->stream);
    comm->io.reset();
  }
  if (comm->nccl) psg::nccl().comm_destroy(comm->nccl);
  delete comm;
}

extern "C" psg_status psg_band_iterate(psg_level* band, psg_comm* comm, int n,
                                       int honor_convergence, psg_iter_stats* stats,
                                       int* n_done) {
  try {
    if (!band || !comm) fail(PSG_E_DOMAIN, "null argument");
    psg_band b{};
    psg_opt_cfg cfg{};
    int C = 0, hist = 0, iter0 = 0;
    psg::band_info(band, &b, &cfg, &C, &hist, &iter0);
    if (b.world != comm->world || b.rank != comm->rank)
      fail(PSG_E_SHAPE, "band plan does not match the communicator's rank / world size");
    psg::StreamScope _ss(comm->ctx->stream);
    if (!comm->io || !comm->io->matches(b, C, cfg, hist != 0)) {
      comm->io = std::make_shared<psg::BandIO>();
      comm->io->setup(b, C, cfg, hist != 0);
    }
    psg::BandIO& io = *comm->io;
    const int64_t total = (int64_t)b.nx * b.ny;
    int done = 0;
    for (int i = 0; i < n; ++i) {
      const bool conv = psg::nccl_iteration(band, comm, io, stats ? stats + i : nullptr,
                                            honor_convergence != 0, total, cfg, iter0 + i + 1);
      ++done;
      if (conv) break;
    }
    if (n_done) *n_done = done;
    return PSG_OK;
  } catch (const psg::Error& e) {
    psg::set_last_error(e.what());
    return e.code;
  } catch (const std::exception& e) {
    psg::set_last_error(e.what());
    return PSG_E_LOGIC;
  }
}

extern "C" psg_status psg_optimize_level_sharded(psg_ctx* ctx, psg_comm* comm,
                                                 const psg_index* index, const double* rows,
                                                 int W, int H, const psg_opt_cfg* cfg,
                                                 const double* ex_hist, double* out_rows,
                                                 psg_iter_stats* stats, int* n_iters) {
  try {
    if (!ctx || !comm || !index || !rows || !cfg || !out_rows) fail(PSG_E_DOMAIN, "null argument");
    psg_band b{};
    psg::check(psg_shard_plan(W, H, psg::index_window(index), cfg->spacing, comm->rank,
                              comm->world, &b));
    psg_level* L = nullptr;
    psg::check(psg_band_create(ctx, index, rows, &b, cfg, ex_hist, &L));
    std::unique_ptr<psg_level, void (*)(psg_level*)> hold(L, psg_level_destroy);
    psg::check(psg_level_prime(L));
    int done = 0;
    psg::check(psg_band_iterate(L, comm, cfg->max_iterations, 1, stats, &done));
    if (n_iters) *n_iters = done;
    psg::check(psg::band_download_owned(L, out_rows));
    return PSG_OK;
  } catch (const psg::Error& e) {
    psg::set_last_error(e.what());
    return e.code;
  }
}

// The same schedule for `world` bands of one image in this process: the
// exchanges are device copies on the context stream (and the histogram sum a
// host reduction); used to test the exchange buffers on one GPU.
extern "C" psg_status psg_optimize_level_loopback(psg_ctx* ctx, const psg_index* index,
                                                  const double* init, int W, int H,
                                                  const psg_opt_cfg* cfg, const double* ex_hist,
                                                  int world, double* out_planes,
                                                  psg_iter_stats* stats, int* n_iters) {
  try {
    if (!ctx || !index || !init || !cfg || !out_planes) fail(PSG_E_DOMAIN, "null argument");
    psg::StreamScope _ss(ctx->stream);
    const int C = psg::index_channels(index), w = psg::index_window(index);
    const size_t P = (size_t)W * H;
    std::vector<psg_band> plans(world);
    for (int r = 0; r < world; ++r)
      psg::check(psg_shard_plan(W, H, w, cfg->spacing, r, world, &plans[r]));
    std::vector<std::unique_ptr<psg_level, void (*)(psg_level*)>> bands;
    std::vector<psg::BandIO> io(world);
    for (int r = 0; r < world; ++r) {
      const psg_band& b = plans[r];
      const int rows = b.e1 - b.p0;
      std::vector<double> part((size_t)C * rows * W);
      for (int c = 0; c < C; ++c)
        std::memcpy(part.data() + (size_t)c * rows * W, init + c * P + (size_t)b.p0 * W,
                    sizeof(double) * rows * W);
      psg_level* L = nullptr;
      psg::check(psg_band_create(ctx, index, part.data(), &b, cfg, ex_hist, &L));
      bands.emplace_back(L, psg_level_destroy);
      psg_band bb{};
      psg_opt_cfg cc{};
      int CC = 0, hist = 0, it0 = 0;
      psg::band_info(L, &bb, &cc, &CC, &hist, &it0);
      io[r].setup(b, C, *cfg, hist != 0);
    }
    for (auto& L : bands) psg::check(psg_level_prime(L.get()));
    const int64_t total = (int64_t)plans[0].nx * plans[0].ny;
    cudaStream_t s = ctx->stream;
    int done = 0;
    for (int it = 1; it <= cfg->max_iterations; ++it) {
      for (int r = 0; r < world; ++r)
        psg::check(psg_band_phase1(bands[r].get(), io[r].hist ? io[r].counts.p : nullptr));
      if (io[0].hist) {  // all-reduce(sum): exact integers
        const size_t nb = io[0].counts.n;
        std::vector<unsigned long long> sum(nb, 0), h(nb);
        for (int r = 0; r < world; ++r) {
          io[r].counts.download(ctx, h.data(), nb);
          PSG_CUDA(cudaStreamSynchronize(s));
          for (size_t k = 0; k < nb; ++k) sum[k] += h[k];
        }
        for (int r = 0; r < world; ++r) io[r].counts_g.upload(ctx, sum.data(), nb);
      }
      for (int r = 0; r < world; ++r)
        psg::check(psg_band_phase2(bands[r].get(), io[r].hist ? io[r].counts_g.p : nullptr,
                                   io[r].send_row0, io[r].send_ae.p));
      for (int r = 1; r < world; ++r)  // rank r receives rank r-1's (eff, idx) rows
        if (io[r].n_halo_ae > 0)
          PSG_CUDA(cudaMemcpyAsync(io[r].recv_ae.p, io[r - 1].send_ae.p, io[r].n_halo_ae * 12,
                                   cudaMemcpyDeviceToDevice, s));
      for (int r = 0; r < world; ++r)
        psg::check(psg_band_phase3(bands[r].get(), io[r].n_halo_ae > 0 ? io[r].recv_ae.p : nullptr,
                                   io[r].n_send_rows,
                                   io[r].n_send_rows > 0 ? io[r].send_rows.p : nullptr));
      for (int r = 0; r + 1 < world; ++r)  // rank r receives rank r+1's first rows
        if (io[r].n_halo_rows > 0)
          PSG_CUDA(cudaMemcpyAsync(io[r].recv_rows.p, io[r + 1].send_rows.p,
                                   sizeof(float) * io[r].n_halo_rows * W * C,
                                   cudaMemcpyDeviceToDevice, s));
      double g[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
      for (int r = 0; r < world; ++r) {
        double p[9];
        psg::check(psg_band_phase4(bands[r].get(),
                                   io[r].n_halo_rows > 0 ? io[r].recv_rows.p : nullptr, p));
        for (int j = 0; j < 9; ++j) g[j] += p[j];
      }
      for (int r = 0; r < world; ++r)
        psg::check(psg_band_commit(bands[r].get(), g, r == 0 && stats ? stats + it - 1 : nullptr));
      ++done;
      if (it >= cfg->min_iterations && g[3] < cfg->convergence_fraction * (double)total) break;
    }
    if (n_iters) *n_iters = done;
    for (int r = 0; r < world; ++r) {
      const psg_band& b = plans[r];
      const int rows = b.p1 - b.p0;
      std::vector<double> own((size_t)C * rows * W);
      psg::check(psg::band_download_owned(bands[r].get(), own.data()));
      for (int c = 0; c < C; ++c)
        std::memcpy(out_planes + c * P + (size_t)b.p0 * W, own.data() + (size_t)c * rows * W,
                    sizeof(double) * rows * W);
    }
    return PSG_OK;
  } catch (const psg::Error& e) {
    psg::set_last_error(e.what());
    return e.code;
  }
}
