// abi.cu — C ABI entry points of libchg (include/chg.h): context, graph and
// model handles, canonical parameter layout, load-balance sampler, NCCL
// bootstrap.  Compute lives in graph.cu / model.cu.
#include <mutex>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <numeric>

#include "common.cuh"
#include "gemm.cuh"

void destroy_graph_impl(chg_graph *G);
void graph_fill_counts(chg_graph *G);
void derivative_impl(chg_ctx *ctx, chg_model *m, chg_graph *g, chg_pred *out);
extern "C" void graph_use(chg_ctx *ctx, chg_graph *g);
void md_verlet(chg_ctx *ctx, int64_t n, double *pos, double *vel, const float *F, const double *inv_mass, double dt,
               int drift);

// ---------------------------------------------------------------------------
// ctx helpers
// ---------------------------------------------------------------------------
void *chg_ctx::get(const std::string &name, size_t bytes) {
  if (bytes == 0) bytes = 16;
  auto it = ws.find(name);
  if (it != ws.end() && it->second.second >= bytes) return it->second.first;
  if (capturing) CHG_THROW(CHG_ERR_STATE, "workspace %s would grow inside a captured step", name.c_str());
  ++ws_gen;
  if (it != ws.end()) CUDA_OK(cudaFreeAsync(it->second.first, stream));
  size_t cap = bytes + bytes / 4 + 256;
  void *p = nullptr;
  CUDA_OK(cudaMallocAsync(&p, cap, stream));
  ws[name] = {p, cap};
  return p;
}

cudaEvent_t chg_ctx::next_event() {
  if (ev_used == ev_pool.size()) {
    cudaEvent_t e;
    CUDA_OK(cudaEventCreate(&e));
    ev_pool.push_back(e);
  }
  return ev_pool[ev_used++];
}

void *chg_ctx::pinned_get(size_t bytes) {
  if (bytes <= pinned_bytes) return pinned;
  CUDA_OK(cudaStreamSynchronize(stream));
  if (pinned) CUDA_OK(cudaFreeHost(pinned));
  size_t cap = std::max<size_t>(bytes * 2, 1 << 20);
  CUDA_OK(cudaMallocHost(&pinned, cap));
  pinned_bytes = cap;
  return pinned;
}

#define ABI_GUARD(ctx, ...)                                     \
  try {                                                         \
    __VA_ARGS__;                                                \
    return CHG_OK;                                              \
  } catch (const ChgError &e) {                                 \
    if (ctx) (ctx)->err = e.msg;                                \
    return e.code;                                              \
  } catch (const std::exception &e) {                           \
    if (ctx) (ctx)->err = e.what();                             \
    return CHG_ERR_ARG;                                         \
  }

// ---------------------------------------------------------------------------
// canonical parameter layout (the library's own table; DESIGN.md lists it and
// tests check it against the oracle's independent table)
// ---------------------------------------------------------------------------
static void build_layout(chg_model *m) {
  const chg_model_cfg &c = m->cfg;
  int d = c.d, h = c.gmlp_hidden, H = c.head_hidden;
  std::vector<std::pair<std::string, std::pair<int, int>>> L;
  auto add = [&](const std::string &n, int r, int k) { L.push_back({n, {r, k}}); };
  add("embed.W", c.n_species, d);
  add("rbf_a.freq", c.n_radial, 0);
  add("rbf_b.freq", c.n_radial, 0);
  add("proj.W0", c.n_radial, d);
  add("proj.Wa", c.n_radial, d);
  add("proj.Wb", c.n_radial, d);
  add("proj.Wtheta", c.n_angular, d);
  auto gmlp = [&](const std::string &pre, int fan, int hid) {
    for (const char *br : {"core", "gate"}) {
      std::string b = pre + "." + br;
      if (hid) {
        add(b + ".W1", fan, hid); add(b + ".b1", hid, 0);
        add(b + ".W2", hid, d);   add(b + ".b2", d, 0);
      } else {
        add(b + ".W", fan, d);    add(b + ".b", d, 0);
      }
    }
    add(pre + ".ln_core.g", d, 0); add(pre + ".ln_core.b", d, 0);
    add(pre + ".ln_gate.g", d, 0); add(pre + ".ln_gate.b", d, 0);
  };
  for (int t = 0; t < c.n_atom_conv; ++t) {
    std::string p = "atom" + std::to_string(t);
    gmlp(p, 3 * d, h);
    add(p + ".out.W", d, d); add(p + ".out.b", d, 0);
  }
  for (int t = 0; t < c.n_bond_conv; ++t) {
    std::string p = "bond" + std::to_string(t);
    gmlp(p, 4 * d, h);
    add(p + ".out.W", d, d); add(p + ".out.b", d, 0);
  }
  for (int t = 0; t < c.n_bond_conv; ++t) gmlp("angle" + std::to_string(t), 4 * d, 0);
  auto mlp = [&](const std::string &pre, std::vector<int> dims) {
    for (size_t k = 0; k + 1 < dims.size(); ++k) {
      add(pre + ".W" + std::to_string(k), dims[k], dims[k + 1]);
      add(pre + ".b" + std::to_string(k), dims[k + 1], 0);
    }
  };
  mlp("head_E", {d, H, H, H, 1});
  add("head_M.W", d, 1); add("head_M.b", 1, 0);
  mlp("head_F", {d, H, H, 1});
  mlp("head_S", {d, H, H, 9});
  int64_t off = 0;
  for (auto &t : L) {
    m->index[t.first] = (int)m->names.size();
    m->names.push_back(t.first);
    m->offsets.push_back(off);
    m->shapes.push_back(t.second.first);
    m->shapes.push_back(t.second.second);
    off += (int64_t)t.second.first * (t.second.second ? t.second.second : 1);
  }
  m->P = off;
  for (auto &n : m->names) m->name_ptrs.push_back(n.c_str());
}

// ---------------------------------------------------------------------------
int device_sm_count() {
  static std::mutex mu;
  static std::map<int, int> cache;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  auto it = cache.find(dev);
  if (it != cache.end()) return it->second;
  int n = 0;
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  cache[dev] = n;
  return n;
}

void smem_optin(const void *func, int bytes) {
  static std::mutex mu;
  static std::map<std::pair<const void *, int>, int> done;   // (kernel, device) -> bytes opted in
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  int &have = done[{func, dev}];
  if (have >= bytes) return;
  CUDA_OK(cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
  have = bytes;
}

extern "C" {

chg_status chg_ctx_create(int device, void *cuda_stream, chg_ctx **out) {
  if (!out) return CHG_ERR_ARG;
  chg_ctx *ctx = new chg_ctx();
  try {
    ctx->device = device;
    CUDA_OK(cudaSetDevice(device));
    if (cuda_stream) {
      ctx->stream = (cudaStream_t)cuda_stream;
    } else {
      CUDA_OK(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
      ctx->own_stream = true;
    }
    // keep freed blocks in the stream-ordered pool (no per-step cudaMalloc)
    cudaMemPool_t pool;
    CUDA_OK(cudaDeviceGetDefaultMemPool(&pool, device));
    uint64_t thr = UINT64_MAX;
    CUDA_OK(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
    CUDA_OK(cudaMalloc(&ctx->d_flag, 256));
    CUDA_OK(cudaMemset(ctx->d_flag, 0, 256));
    CUDA_OK(cudaMallocHost(&ctx->h_flags, sizeof(int) * chg_ctx::NFLAG));
    for (int i = 0; i < chg_ctx::NFLAG; ++i) ctx->h_flags[i] = 0x7f7f7f7f;
    ctx->d_loss = (double *)((char *)ctx->d_flag + 64);
  } catch (const ChgError &e) {
    delete ctx;
    return e.code;
  }
  *out = ctx;
  return CHG_OK;
}

void chg_ctx_destroy(chg_ctx *ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  for (auto &kv : ctx->ws) cudaFree(kv.second.first);
  if (ctx->pinned) cudaFreeHost(ctx->pinned);
  if (ctx->d_flag) cudaFree(ctx->d_flag);
  if (ctx->h_flags) cudaFreeHost(ctx->h_flags);
  for (auto &p : ctx->pending) cudaEventDestroy(p.ev);
  for (auto e : ctx->flag_ev_pool) cudaEventDestroy(e);
  if (ctx->nccl_comm) ncclCommDestroy((ncclComm_t)ctx->nccl_comm);
  for (auto e : ctx->ev_pool) cudaEventDestroy(e);
  if (ctx->side) cudaStreamDestroy(ctx->side);
  if (ctx->comm) cudaStreamDestroy(ctx->comm);
  if (ctx->ev_comm_in) cudaEventDestroy(ctx->ev_comm_in);
  if (ctx->ev_comm_done) cudaEventDestroy(ctx->ev_comm_done);
  if (ctx->ev_fork) cudaEventDestroy(ctx->ev_fork);
  if (ctx->ev_join) cudaEventDestroy(ctx->ev_join);
  if (ctx->own_stream) cudaStreamDestroy(ctx->stream);
  delete ctx;
}

const char *chg_last_error(const chg_ctx *ctx) { return ctx ? ctx->err.c_str() : "null ctx"; }

chg_status chg_sync(chg_ctx *ctx) {
  if (!ctx) return CHG_ERR_ARG;
  ABI_GUARD(ctx, {
    CUDA_OK(cudaStreamSynchronize(ctx->stream));
    CUDA_OK(cudaGetLastError());
    check_pending(ctx, true);
  });
}

int64_t chg_launch_count(const chg_ctx *ctx) { return ctx ? ctx->launches : -1; }

chg_status chg_nccl_unique_id(void *uid128) {
  if (!uid128) return CHG_ERR_ARG;
  ncclUniqueId id;
  if (ncclGetUniqueId(&id) != ncclSuccess) return CHG_ERR_NCCL;
  static_assert(sizeof(ncclUniqueId) == 128, "nccl uid size");
  memcpy(uid128, &id, 128);
  return CHG_OK;
}

chg_status chg_ctx_set_nccl(chg_ctx *ctx, const void *uid128, int nranks, int rank) {
  if (!ctx || !uid128 || nranks < 1 || rank < 0 || rank >= nranks) return CHG_ERR_ARG;
  ABI_GUARD(ctx, {
    CUDA_OK(cudaSetDevice(ctx->device));
    ncclUniqueId id;
    memcpy(&id, uid128, 128);
    ncclComm_t comm;
    ncclResult_t r = ncclCommInitRank(&comm, nranks, id, rank);
    if (r != ncclSuccess) CHG_THROW(CHG_ERR_NCCL, "ncclCommInitRank: %s", ncclGetErrorString(r));
    if (ctx->nccl_comm) ncclCommDestroy((ncclComm_t)ctx->nccl_comm);
    ctx->nccl_comm = comm;
    ctx->nranks = nranks;
    ctx->rank = rank;
  });
}

chg_status chg_ctx_set_grad_overlap(chg_ctx *ctx, int on) {
  if (!ctx) return CHG_ERR_ARG;
  ctx->grad_overlap = on != 0;
  return CHG_OK;
}

chg_status chg_build_graph(chg_ctx *ctx, int32_t n_struct, const int64_t *atom_ptr, const double *positions,
                           const double *lattice, const int32_t *species, chg_cutoffs cutoffs,
                           int inputs_on_device, chg_graph **out) {
  if (!ctx || !out) return CHG_ERR_ARG;
  ABI_GUARD(ctx, {
    CUDA_OK(cudaSetDevice(ctx->device));
    *out = build_graph_impl(ctx, n_struct, atom_ptr, positions, lattice, species, cutoffs.r_atom,
                            cutoffs.r_bond, inputs_on_device, 94);
  });
}

chg_status chg_build_graph_skin(chg_ctx *ctx, int32_t n_struct, const int64_t *atom_ptr, const double *positions,
                                const double *lattice, const int32_t *species, chg_cutoffs cutoffs, double skin,
                                int inputs_on_device, chg_graph **out) {
  if (!ctx || !out) return CHG_ERR_ARG;
  ABI_GUARD(ctx, {
    CUDA_OK(cudaSetDevice(ctx->device));
    *out = build_graph_impl(ctx, n_struct, atom_ptr, positions, lattice, species, cutoffs.r_atom,
                            cutoffs.r_bond, inputs_on_device, 94, skin);
  });
}

chg_status chg_graph_refresh(chg_ctx *ctx, chg_graph *g, const double *positions, int32_t *flag) {
  if (!ctx || !g || (g->N > 0 && !positions)) return CHG_ERR_ARG;
  ABI_GUARD(ctx, {
    CUDA_OK(cudaSetDevice(ctx->device));
    graph_use(ctx, g);
    graph_refresh(ctx, g, positions, flag);
  });
}

chg_status chg_graph_counts(const chg_graph *g, int64_t tot[4], int64_t *per_struct) {
  if (!g || !tot) return CHG_ERR_ARG;
  tot[0] = g->N; tot[1] = g->E; tot[2] = g->B; tot[3] = g->A;
  if (per_struct) {
    chg_graph *G = const_cast<chg_graph *>(g);    // lazily cached host copy (logically const)
    if (!G->counts_ready) {
      try {
        graph_fill_counts(G);
      } catch (const ChgError &e) {
        G->ctx->err = e.msg;
        return e.code;
      }
    }
    std::copy(g->counts_h.begin(), g->counts_h.end(), per_struct);
  }
  return CHG_OK;
}

chg_status chg_graph_export(const chg_graph *g, int32_t *row_ptr, int32_t *nbr, int8_t *img, float *vec,
                            int32_t *bond_id, int32_t *bond_edge, int32_t *angle_ptr, int32_t *angle_b1,
                            int32_t *angle_b2, int32_t *rev, int32_t *swap) {
  if (!g) return CHG_ERR_ARG;
  chg_ctx *ctx = g->ctx;
  ABI_GUARD(ctx, {
    cudaStream_t st = ctx->stream;
    auto cp = [&](void *dst, const void *src, size_t bytes) {
      if (dst && bytes) CUDA_OK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, st));
    };
    cp(row_ptr, g->row_ptr, 4 * (g->N + 1));
    cp(nbr, g->nbr, 4 * g->E);
    cp(vec, g->vec, 16 * g->E);
    cp(bond_id, g->bond_id, 4 * g->E);
    cp(bond_edge, g->bond_edge, 4 * g->B);
    cp(angle_ptr, g->angle_ptr, 4 * (g->B + 1));
    cp(angle_b1, g->angle_b1, 4 * g->A);
    cp(angle_b2, g->angle_b2, 4 * g->A);
    cp(rev, g->rev, 4 * g->E);
    cp(swap, g->swap, 4 * g->A);
    std::vector<char4> tmp(img ? g->E : 0);
    if (img && g->E) cp(tmp.data(), g->img, 4 * g->E);
    CUDA_OK(cudaStreamSynchronize(st));
    for (int64_t e = 0; e < (int64_t)tmp.size(); ++e) {
      img[3 * e] = tmp[e].x; img[3 * e + 1] = tmp[e].y; img[3 * e + 2] = tmp[e].z;
    }
  });
}

void chg_graph_destroy(chg_graph *g) { destroy_graph_impl(g); }

chg_status chg_model_create(chg_ctx *ctx, const chg_model_cfg *cfg, chg_model **out) {
  if (!ctx || !cfg || !out) return CHG_ERR_ARG;
  chg_model *m = new chg_model();
  try {
    m->ctx = ctx;
    m->cfg = *cfg;
    const chg_model_cfg &c = *cfg;
    if (c.d != 64 || c.n_radial != 31 || c.n_angular != 31 || c.gmlp_hidden != 64 || c.head_hidden != 64 ||
        c.n_atom_conv != c.n_bond_conv + 1 || c.n_bond_conv < 1 || c.n_species != 94 || c.envelope_p < 2 ||
        c.mlp_precision < 0 || c.mlp_precision > 3)
      CHG_THROW(CHG_ERR_ARG, "unsupported model config (built: d=64, K=31, hidden 64, n_atom_conv = n_bond_conv+1, "
                             "94 species, mlp_precision 0 (fp32), 1 (3xTF32 tcgen05), 2 (TF32 tcgen05) or 3 (BF16 tcgen05))");
    build_layout(m);
    CUDA_OK(cudaSetDevice(ctx->device));
    // params | grads | adam m | adam v, each segment 256-B aligned (vector loads and stores)
    const int64_t Ps = (m->P + 63) & ~(int64_t)63;
    CUDA_OK(cudaMalloc(&m->params, 4 * Ps * 4));
    m->grads = m->params + Ps;
    m->m = m->params + 2 * Ps;
    m->v = m->params + 3 * Ps;
    CUDA_OK(cudaMemset(m->params, 0, 4 * Ps * 4));
    std::vector<int64_t> toff;
    std::vector<int32_t> trc;
    for (size_t t = 0; t < m->names.size(); ++t) {
      if (m->shapes[2 * t + 1] == 0) continue;
      toff.push_back(m->offsets[t]);
      trc.push_back(m->shapes[2 * t]);
      trc.push_back(m->shapes[2 * t + 1]);
    }
    m->n2d = (int)toff.size();
    CUDA_OK(cudaMalloc(&m->d_toff, 8 * toff.size() + 4 * trc.size()));
    m->d_trc = (int32_t *)(m->d_toff + toff.size());
    CUDA_OK(cudaMemcpy(m->d_toff, toff.data(), 8 * toff.size(), cudaMemcpyHostToDevice));
    CUDA_OK(cudaMemcpy(m->d_trc, trc.data(), 4 * trc.size(), cudaMemcpyHostToDevice));
  } catch (const ChgError &e) {
    ctx->err = e.msg;
    delete m;
    return e.code;
  }
  *out = m;
  return CHG_OK;
}

void chg_model_destroy(chg_model *m) {
  if (!m) return;
  cudaSetDevice(m->ctx->device);
  cudaStreamSynchronize(m->ctx->stream);
  for (auto &p : m->ctx->pending)                  // deferred checks of this model report no name
    if (p.m == m) p.m = nullptr;
  cudaFree(m->params);
  if (m->d_toff) cudaFree(m->d_toff);
  tc_cache_free(m);
  if (m->wt) cudaFree(m->wt);
  delete m;
}

chg_status chg_model_layout(const chg_model *m, int *n, const char *const **names, const int64_t **offsets,
                            const int32_t **shapes) {
  if (!m || !n) return CHG_ERR_ARG;
  *n = (int)m->names.size();
  if (names) *names = m->name_ptrs.data();
  if (offsets) *offsets = m->offsets.data();
  if (shapes) *shapes = m->shapes.data();
  return CHG_OK;
}

int64_t chg_model_num_params(const chg_model *m) { return m ? m->P : -1; }

static float *which_ptr(const chg_model *m, int which) {
  switch (which) {
    case 0: return m->params;
    case 1: return m->grads;
    case 2: return m->m;
    case 3: return m->v;
  }
  return nullptr;
}

chg_status chg_model_set(chg_model *m, int which, const float *host, int64_t n) {
  if (!m || !host || n != m->P || !which_ptr(m, which)) return CHG_ERR_ARG;
  ABI_GUARD(m->ctx, {
    CUDA_OK(cudaMemcpyAsync(which_ptr(m, which), host, 4 * n, cudaMemcpyHostToDevice, m->ctx->stream));
    CUDA_OK(cudaStreamSynchronize(m->ctx->stream));
  });
}

chg_status chg_model_get(const chg_model *m, int which, float *host, int64_t n) {
  if (!m || !host || n != m->P || !which_ptr(m, which)) return CHG_ERR_ARG;
  ABI_GUARD(m->ctx, {
    CUDA_OK(cudaMemcpyAsync(host, which_ptr(m, which), 4 * n, cudaMemcpyDeviceToHost, m->ctx->stream));
    CUDA_OK(cudaStreamSynchronize(m->ctx->stream));
  });
}

void *chg_model_device_ptr(chg_model *m, int which) { return m ? which_ptr(m, which) : nullptr; }

// a graph built by another context (e.g. a prefetching builder) of the same device: this
// context's stream waits for the build; the graph frees its arrays after this stream's work
void graph_use(chg_ctx *ctx, chg_graph *g) {
  if (g->ctx == ctx) return;
  if (g->ctx->device != ctx->device) CHG_THROW(CHG_ERR_ARG, "graph built on device %d, used on %d", g->ctx->device, ctx->device);
  if (g->user && g->user != ctx) CHG_THROW(CHG_ERR_ARG, "graph already used by a third context");
  CUDA_OK(cudaStreamWaitEvent(ctx->stream, g->ready, 0));
  g->user = ctx;
}

chg_status chg_graph_wait(chg_ctx *ctx, chg_graph *g) {
  if (!ctx || !g) return CHG_ERR_ARG;
  ABI_GUARD(ctx, {
    CUDA_OK(cudaSetDevice(ctx->device));
    graph_use(ctx, g);
  });
}

chg_status chg_forward(chg_ctx *ctx, chg_model *m, chg_graph *g, int train, chg_pred *out) {
  if (!ctx || !m || !g) return CHG_ERR_ARG;
  if (m->ctx != ctx) { ctx->err = "model bound to another ctx"; return CHG_ERR_ARG; }
  ABI_GUARD(ctx, {
    CUDA_OK(cudaSetDevice(ctx->device));
    graph_use(ctx, g);
    forward_impl(ctx, m, g, train, out);
  });
}

chg_status chg_forward_conservative(chg_ctx *ctx, chg_model *m, chg_graph *g, chg_pred *out) {
  if (!ctx || !m || !g) return CHG_ERR_ARG;
  if (m->ctx != ctx) { ctx->err = "model bound to another ctx"; return CHG_ERR_ARG; }
  ABI_GUARD(ctx, {
    CUDA_OK(cudaSetDevice(ctx->device));
    graph_use(ctx, g);
    derivative_impl(ctx, m, g, out);
  });
}

chg_status chg_md_verlet(chg_ctx *ctx, int64_t n_atoms, double *positions, double *velocities, const float *forces,
                         const double *inv_mass, double dt_fs, int drift) {
  if (!ctx || n_atoms < 0 || (n_atoms > 0 && (!positions || !velocities || !forces || !inv_mass))) return CHG_ERR_ARG;
  ABI_GUARD(ctx, {
    CUDA_OK(cudaSetDevice(ctx->device));
    md_verlet(ctx, n_atoms, positions, velocities, forces, inv_mass, dt_fs, drift);
  });
}

chg_status chg_backward(chg_ctx *ctx, chg_model *m, chg_graph *g, const chg_labels *labels,
                        const chg_loss_cfg *cfg, double loss_out[5]) {
  if (!ctx || !m || !g || !labels || !cfg) return CHG_ERR_ARG;
  if (!ctx->fwd_train || ctx->fwd_graph != g || ctx->fwd_graph_id != g->id) {
    ctx->err = "chg_backward needs a train-mode chg_forward on the same graph first";
    return CHG_ERR_STATE;
  }
  ABI_GUARD(ctx, {
    CUDA_OK(cudaSetDevice(ctx->device));
    backward_impl(ctx, m, g, labels, cfg, loss_out);
  });
}

chg_status chg_step(chg_ctx *ctx, chg_model *m, const chg_adam_cfg *cfg) {
  if (!ctx || !m || !cfg) return CHG_ERR_ARG;
  ABI_GUARD(ctx, {
    CUDA_OK(cudaSetDevice(ctx->device));
    step_impl(ctx, m, cfg, -1);
  });
}

chg_status chg_balance(const int64_t *loads, int32_t n, int32_t n_ranks, int32_t *rank_of) {
  if (n_ranks <= 0 || n < 0 || (n > 0 && (!loads || !rank_of))) return CHG_ERR_ARG;
  std::vector<int32_t> order(n);
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(), [&](int32_t a, int32_t b) { return loads[a] < loads[b]; });
  int lo = 0, hi = n - 1, turn = 0;
  while (lo <= hi) {
    int r = turn % n_ranks;
    rank_of[order[lo++]] = r;
    if (lo <= hi) rank_of[order[hi--]] = r;
    ++turn;
  }
  return CHG_OK;
}

chg_status chg_profile(chg_ctx *ctx, int mode) {
  if (!ctx) return CHG_ERR_ARG;
  ABI_GUARD(ctx, {
    if (mode == 0 || mode == 1) {
      CUDA_OK(cudaStreamSynchronize(ctx->stream));
      ctx->prof.clear();
      ctx->ev_used = 0;
      ctx->prof_on = mode == 1;
    } else {
      CHG_THROW(CHG_ERR_ARG, "mode must be 0 or 1");
    }
  });
}

chg_status chg_profile_query(chg_ctx *ctx, int idx, char *tag, double *ms, int64_t *launches, double *flops,
                             double *bytes) {
  if (!ctx || idx < 0) return CHG_ERR_ARG;
  ABI_GUARD(ctx, {
    CUDA_OK(cudaStreamSynchronize(ctx->stream));
    std::vector<std::string> tags;
    for (auto &r : ctx->prof)
      if (std::find(tags.begin(), tags.end(), std::string(r.tag)) == tags.end()) tags.push_back(r.tag);
    if (idx >= (int)tags.size()) CHG_THROW(CHG_ERR_ARG, "no profile entry %d", idx);
    double t = 0, f = 0, b = 0;
    int64_t n = 0;
    for (auto &r : ctx->prof) {
      if (tags[idx] != r.tag) continue;
      float e = 0;
      CUDA_OK(cudaEventElapsedTime(&e, ctx->ev_pool[r.ev], ctx->ev_pool[r.ev + 1]));
      t += e; f += r.flops; b += r.bytes; ++n;
    }
    if (tag) { strncpy(tag, tags[idx].c_str(), 63); tag[63] = 0; }
    if (ms) *ms = t;
    if (launches) *launches = n;
    if (flops) *flops = f;
    if (bytes) *bytes = b;
  });
}

chg_status chg_debug_get(chg_ctx *ctx, const char *name, float *host, int64_t n, int64_t *rows, int64_t *cols) {
  if (!ctx || !name) return CHG_ERR_ARG;
  ABI_GUARD(ctx, {
    auto it = ctx->dbg.find(name);
    if (it == ctx->dbg.end()) CHG_THROW(CHG_ERR_ARG, "no debug tensor '%s'", name);
    const auto &d = it->second;
    if (rows) *rows = d.rows;
    if (cols) *cols = d.cols;
    if (host) {
      if (n < d.rows * d.cols) CHG_THROW(CHG_ERR_ARG, "buffer too small");
      if (d.rows * d.cols)
        CUDA_OK(cudaMemcpy2DAsync(host, 4 * d.cols, d.p, 4 * d.ld, 4 * d.cols, d.rows, cudaMemcpyDeviceToHost,
                                  ctx->stream));
      CUDA_OK(cudaStreamSynchronize(ctx->stream));
    }
  });
}

}  // extern "C"
