// capture.cu — one training step (forward + backward + [allreduce] + finite check + Adam) as a
// CUDA graph (chg_capture_step / chg_exec_step, include/chg.h).
//
// The step's ~140 launches are recorded once per (model, graph) and replayed with one
// cudaGraphLaunch: no per-launch host work, no host synchronisation inside the step (labels on
// the device, loss not read back, the finite flag copied to a pinned slot and checked by a
// later call).  The only per-step host work is updating the Adam node's scalars (lr, bias
// corrections) in the instantiated graph.
#include <cmath>

#include "gemm.cuh"
#include "ops.cuh"

extern "C" void graph_use(chg_ctx *ctx, chg_graph *g);   // abi.cu
void derivative_impl(chg_ctx *ctx, chg_model *m, chg_graph *g, chg_pred *out);   // model.cu

struct chg_exec {
  chg_ctx *ctx = nullptr;
  chg_model *m = nullptr;
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  cudaGraphNode_t adam = nullptr;      // the k_adam kernel node
  cudaKernelNodeParams adam_params{};
  uint64_t ws_gen = 0;
  int slot = 0;                        // pinned finite-flag slot written by every replay
  int64_t launches = 0;                // kernels per replay (bookkeeping)
  int64_t n = 0;
  float *p = nullptr, *g = nullptr, *mm = nullptr, *v = nullptr;
  const int *bad = nullptr;
};

namespace {

void set_adam_args(chg_exec *x, const chg_adam_cfg *cfg) {
  const double bc1 = 1.0 - std::pow((double)cfg->beta1, (double)cfg->step);
  const double bc2 = 1.0 - std::pow((double)cfg->beta2, (double)cfg->step);
  float lr = cfg->lr, b1 = cfg->beta1, b2 = cfg->beta2, eps = cfg->eps;
  float step_size = (float)(lr / bc1), inv_sqrt_bc2 = (float)(1.0 / std::sqrt(bc2));
  // k_adam(n, p, g, m, v, lr, b1, b2, eps, step_size, inv_sqrt_bc2, bad)
  void *args[12] = {&x->n, &x->p, &x->g, &x->mm, &x->v, &lr, &b1, &b2, &eps, &step_size, &inv_sqrt_bc2,
                    (void *)&x->bad};
  cudaKernelNodeParams kp = x->adam_params;
  kp.kernelParams = args;
  kp.extra = nullptr;
  CUDA_OK(cudaGraphExecKernelNodeSetParams(x->exec, x->adam, &kp));
}

}  // namespace

extern "C" {

chg_status chg_capture_step(chg_ctx *ctx, chg_model *m, chg_graph *g, const chg_labels *labels,
                            const chg_loss_cfg *loss, const chg_adam_cfg *adam, chg_exec **out) {
  if (!ctx || !m || !g || !labels || !loss || !adam || !out) return CHG_ERR_ARG;
  if (m->ctx != ctx) { ctx->err = "model bound to another ctx"; return CHG_ERR_ARG; }
  if (!labels->on_device) { ctx->err = "chg_capture_step needs device labels (on_device = 1)"; return CHG_ERR_ARG; }
  if (adam->step < 1) { ctx->err = "adam step must be >= 1"; return CHG_ERR_ARG; }
  chg_exec *x = new chg_exec();
  bool began = false;
  try {
    CUDA_OK(cudaSetDevice(ctx->device));
    graph_use(ctx, g);
    check_pending(ctx, false);
    // 1. one real forward + backward: every workspace reaches its size, every weight image and
    //    tensor map of the call sites exists; the gradients are restored afterwards
    float *gsave = ctx->getf("capture_gsave", (size_t)std::max<int64_t>(m->P, 1));
    CUDA_OK(cudaMemcpyAsync(gsave, m->grads, 4 * (size_t)m->P, cudaMemcpyDeviceToDevice, ctx->stream));
    forward_impl(ctx, m, g, 1, nullptr);
    backward_impl(ctx, m, g, labels, loss, nullptr);
    CUDA_OK(cudaMemcpyAsync(m->grads, gsave, 4 * (size_t)m->P, cudaMemcpyDeviceToDevice, ctx->stream));
    if (ctx->use_tc) tc_repack_all(ctx, m);        // uploads the image table of new call sites (host copy)
    CUDA_OK(cudaStreamSynchronize(ctx->stream));
    // 2. capture the step
    x->ctx = ctx; x->m = m;
    x->slot = next_flag_slot(ctx);
    const int64_t l0 = ctx->launches;
    cudaGetLastError();                              // a stale (already reported) error must not fail the capture
    CUDA_OK(cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal));
    began = true;
    ctx->capturing = true;
    forward_impl(ctx, m, g, 1, nullptr);
    backward_impl(ctx, m, g, labels, loss, nullptr);
    step_impl(ctx, m, adam, x->slot);
    ctx->capturing = false;
    began = false;
    CUDA_OK(cudaStreamEndCapture(ctx->stream, &x->graph));
    x->launches = ctx->launches - l0;
    ctx->launches = l0;
    CUDA_OK(cudaGraphInstantiate(&x->exec, x->graph, 0));
    // 3. the Adam node, whose scalars change every step
    size_t nn = 0;
    CUDA_OK(cudaGraphGetNodes(x->graph, nullptr, &nn));
    std::vector<cudaGraphNode_t> nodes(nn);
    CUDA_OK(cudaGraphGetNodes(x->graph, nodes.data(), &nn));
    for (auto nd : nodes) {
      cudaGraphNodeType t;
      CUDA_OK(cudaGraphNodeGetType(nd, &t));
      if (t != cudaGraphNodeTypeKernel) continue;
      cudaKernelNodeParams kp{};
      if (cudaGraphKernelNodeGetParams(nd, &kp) != cudaSuccess) continue;
      if (kp.func == adam_kernel()) { x->adam = nd; x->adam_params = kp; }
    }
    if (!x->adam) CHG_THROW(CHG_ERR_STATE, "captured step has no Adam node");
    x->n = m->P; x->p = m->params; x->g = m->grads; x->mm = m->m; x->v = m->v; x->bad = ctx->d_flag;
    x->ws_gen = ctx->ws_gen;
    ctx->fwd_train = false;                        // the captured forward's activations are not "live"
    *out = x;
    return CHG_OK;
  } catch (const ChgError &e) {
    ctx->capturing = false;
    if (began) {
      cudaGraph_t junk = nullptr;
      cudaStreamEndCapture(ctx->stream, &junk);
      if (junk) cudaGraphDestroy(junk);
    }
    cudaGetLastError();
    ctx->err = e.msg;
    chg_exec_destroy(x);
    return e.code;
  }
}

chg_status chg_exec_step(chg_ctx *ctx, chg_exec *x, const chg_adam_cfg *adam) {
  if (!ctx || !x || !adam || x->ctx != ctx) return CHG_ERR_ARG;
  try {
    CUDA_OK(cudaSetDevice(ctx->device));
    if (adam->step < 1) CHG_THROW(CHG_ERR_ARG, "adam step must be >= 1");
    if (x->ws_gen != ctx->ws_gen)
      CHG_THROW(CHG_ERR_STATE, "a ctx workspace was re-allocated after this step was captured: capture again");
    check_pending(ctx, false);
    set_adam_args(x, adam);
    CUDA_OK(cudaGraphLaunch(x->exec, ctx->stream));
    ctx->launches += x->launches;
    push_pending(ctx, x->slot, x->m);
    return CHG_OK;
  } catch (const ChgError &e) {
    ctx->err = e.msg;
    return e.code;
  }
}

// ---------------------------------------------------------------------------
// captured MD step (skin graph): kick + drift, geometry refresh, conservative forces, kick
// ---------------------------------------------------------------------------
struct chg_md_exec {
  chg_ctx *ctx = nullptr;
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  uint64_t ws_gen = 0;
  int64_t launches = 0;
};

chg_status chg_md_capture(chg_ctx *ctx, chg_model *m, chg_graph *g, double *pos, double *vel, const double *inv_mass,
                          double dt, const chg_pred *out, int32_t *flag, chg_md_exec **xo) {
  if (!ctx || !m || !g || !out || !xo || (g->N > 0 && (!pos || !vel || !inv_mass || !out->forces))) return CHG_ERR_ARG;
  if (m->ctx != ctx) { ctx->err = "model bound to another ctx"; return CHG_ERR_ARG; }
  if (!out->on_device) { ctx->err = "chg_md_capture needs device outputs (on_device = 1)"; return CHG_ERR_ARG; }
  chg_md_exec *x = new chg_md_exec();
  bool began = false;
  try {
    CUDA_OK(cudaSetDevice(ctx->device));
    graph_use(ctx, g);
    chg_pred o = *out;
    // one real pass: sizes every workspace / weight image, and out->forces = F(current positions)
    derivative_impl(ctx, m, g, &o);
    if (ctx->use_tc) tc_repack_all(ctx, m);
    CUDA_OK(cudaStreamSynchronize(ctx->stream));
    x->ctx = ctx;
    const int64_t l0 = ctx->launches;
    cudaGetLastError();
    CUDA_OK(cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal));
    began = true;
    ctx->capturing = true;
    md_verlet(ctx, g->N, pos, vel, out->forces, inv_mass, dt, 1);
    graph_refresh(ctx, g, pos, flag);
    derivative_impl(ctx, m, g, &o);
    md_verlet(ctx, g->N, pos, vel, out->forces, inv_mass, dt, 0);
    ctx->capturing = false;
    began = false;
    CUDA_OK(cudaStreamEndCapture(ctx->stream, &x->graph));
    x->launches = ctx->launches - l0;
    ctx->launches = l0;
    CUDA_OK(cudaGraphInstantiate(&x->exec, x->graph, 0));
    x->ws_gen = ctx->ws_gen;
    *xo = x;
    return CHG_OK;
  } catch (const ChgError &e) {
    ctx->capturing = false;
    if (began) {
      cudaGraph_t junk = nullptr;
      cudaStreamEndCapture(ctx->stream, &junk);
      if (junk) cudaGraphDestroy(junk);
    }
    cudaGetLastError();
    ctx->err = e.msg;
    chg_md_exec_destroy(x);
    return e.code;
  }
}

chg_status chg_md_run(chg_ctx *ctx, chg_md_exec *x, int n_steps) {
  if (!ctx || !x || x->ctx != ctx || n_steps < 0) return CHG_ERR_ARG;
  try {
    CUDA_OK(cudaSetDevice(ctx->device));
    if (x->ws_gen != ctx->ws_gen)
      CHG_THROW(CHG_ERR_STATE, "a ctx workspace was re-allocated after this MD step was captured: capture again");
    for (int k = 0; k < n_steps; ++k) CUDA_OK(cudaGraphLaunch(x->exec, ctx->stream));
    ctx->launches += x->launches * n_steps;
    return CHG_OK;
  } catch (const ChgError &e) {
    ctx->err = e.msg;
    return e.code;
  }
}

void chg_md_exec_destroy(chg_md_exec *x) {
  if (!x) return;
  if (x->ctx) cudaStreamSynchronize(x->ctx->stream);
  if (x->exec) cudaGraphExecDestroy(x->exec);
  if (x->graph) cudaGraphDestroy(x->graph);
  delete x;
}

void chg_exec_destroy(chg_exec *x) {
  if (!x) return;
  if (x->ctx) cudaStreamSynchronize(x->ctx->stream);
  if (x->exec) cudaGraphExecDestroy(x->exec);
  if (x->graph) cudaGraphDestroy(x->graph);
  delete x;
}

}  // extern "C"
