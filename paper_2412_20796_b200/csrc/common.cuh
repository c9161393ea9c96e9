// common.cuh — internal types and helpers of libchg (FastCHGNet training step, sm_100a).
// Not part of the ABI; see include/chg.h for the public contract.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <map>
#include <string>
#include <vector>

#include "../../include/chg.h"

#define CHG_D 64          // feature width
#define CHG_K 31          // radial / angular basis size
#define CHG_KP 32         // padded basis row stride

// ---------------------------------------------------------------------------
// error handling: C++ exception inside the library, converted at the ABI edge
// ---------------------------------------------------------------------------
struct ChgError {
  chg_status code;
  std::string msg;
};

#define CHG_THROW(code, ...)                                   \
  do {                                                         \
    char _b[512];                                              \
    snprintf(_b, sizeof(_b), __VA_ARGS__);                     \
    throw ChgError{code, std::string(_b)};                     \
  } while (0)

#define CUDA_OK(x)                                                                       \
  do {                                                                                   \
    cudaError_t _e = (x);                                                                \
    if (_e != cudaSuccess)                                                               \
      CHG_THROW(CHG_ERR_CUDA, "%s:%d %s: %s", __FILE__, __LINE__, #x, cudaGetErrorString(_e)); \
  } while (0)

// ---------------------------------------------------------------------------
// deferred split reductions (reduce.cu): every "sum the per-CTA partials into a gradient"
// step of a backward layer is recorded and executed by ONE launch at the layer's end
// ---------------------------------------------------------------------------
struct RedJob {
  int kind = 0;                 // 0 weight gradient (W/b by 64-col chunk), 1 flat, 2 LayerNorm (4 x 64), 3 projection
  int n = 0;                    // outputs
  int splits = 0;               // partial rows
  int64_t stride = 0;           // floats between partial rows
  const float *part = nullptr;  // [splits][stride]
  int K = 0, N = 0;             // kind 0: rows < K -> W, row K -> bias; kind 3: N = columns C
  float *W[4] = {nullptr, nullptr, nullptr, nullptr};
  int ldw[4] = {0, 0, 0, 0};
  float *b[4] = {nullptr, nullptr, nullptr, nullptr};
  int k0[4] = {0, 0, 0, 0}, kn[4] = {-1, -1, -1, -1};
  int block0 = 0;               // first block of this job in the batched launch
  int qpb = 32;                 // float4 quads per block (set by red_flush from n and splits)
};

// ---------------------------------------------------------------------------
// context
// ---------------------------------------------------------------------------
struct chg_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  // second stream for the concurrent bond-conv branch of a forward layer (Eq. 11 makes the
  // atom and bond/angle updates of a layer independent)
  cudaStream_t side = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  // the branches run concurrently unless per-op profiling is on (profiled passes are serial so
  // that every op's CUDA-event time is its own)
  bool concurrent() const { return side != nullptr && !prof_on; }
  std::string err;
  int64_t launches = 0;
  // named device workspaces (grow-only, stream-ordered reallocation)
  std::map<std::string, std::pair<void *, size_t>> ws;
  // pinned host staging
  void *pinned = nullptr;
  size_t pinned_bytes = 0;
  // NCCL
  void *nccl_comm = nullptr;
  int nranks = 1, rank = 0;
  // NEXT-3: gradient allreduce in buckets issued during the backward on `comm`, as soon
  // as a layer's gradients are final; chg_step then only waits for them (ev_comm)
  bool grad_overlap = false;
  cudaStream_t comm = nullptr;
  cudaEvent_t ev_comm_in = nullptr, ev_comm_done = nullptr;
  bool ar_pending = false;
  int ar_buckets = 0;                           // buckets issued by the last backward (bookkeeping)
  // forward bookkeeping for backward
  const chg_graph *fwd_graph = nullptr;
  uint64_t fwd_graph_id = 0;
  bool fwd_train = false;
  // GEMM engine for the current call: false = fp32 CUDA cores, true = tcgen05 (TF32, 3xTF32
  // split operands when tc_split: mlp_precision 1, BF16 operands when tc_bf16: mlp_precision 3)
  bool use_tc = false;
  bool tc_split = false;
  bool tc_bf16 = false;
  void set_precision(int mlp_precision) {
    use_tc = mlp_precision >= 1 && mlp_precision <= 3;
    tc_split = mlp_precision == 1;
    tc_bf16 = mlp_precision == 3;
  }
  // producers may write tensor-core-only operands already TF32-rounded (plain TF32 mode only)
  bool tc_round() const { return use_tc && !tc_split && !tc_bf16; }
  bool forked = false;           // a side-stream branch is in flight: plain launches (no PDL)
  const struct chg_model *cur_model = nullptr;   // model of the current forward/backward
  const float *cur_wt = nullptr;                 // its transposed weight copy (same flat offsets)
  // debug name -> (ptr, rows, cols, ld)
  struct Dbg { const float *p; int64_t rows, cols, ld; };
  std::map<std::string, Dbg> dbg;
  // device scratch for flags / loss
  int *d_flag = nullptr;
  double *d_loss = nullptr;
  // finite flags of chg_step copied to pinned host slots; a deferred check (defer_check or a
  // captured step) is resolved by a later call once its event has completed
  static constexpr int NFLAG = 64;
  int *h_flags = nullptr;                       // pinned [NFLAG]
  int flag_next = 0;
  struct Pending { cudaEvent_t ev; int slot; const struct chg_model *m; };
  std::vector<Pending> pending;
  std::vector<cudaEvent_t> flag_ev_pool;
  // CUDA-graph capture of a training step (chg_capture_step): no workspace may grow while
  // capturing; every (re)allocation bumps ws_gen so stale captures are refused
  bool capturing = false;
  uint64_t ws_gen = 0;

  // optional per-op device timing (chg_profile_*): CUDA events on the ctx stream
  struct ProfRec { const char *tag; int ev; double flops, bytes; };
  bool prof_on = false;
  std::vector<ProfRec> prof;
  std::vector<cudaEvent_t> ev_pool;
  size_t ev_used = 0;
  cudaEvent_t next_event();

  // scratch shared by kernels that may run on either stream gets a per-stream name
  std::string ws_name(const char *base) const { return stream == side && side ? std::string(base) + "#side" : base; }
  // deferred reductions (reduce.cu): active inside backward layers
  bool red_on = false;
  // conservative-force pass (deriv.cu): the backward runs without parameter gradients
  bool no_param_grads = false;
  std::vector<RedJob> red_jobs;
  void *get(const std::string &name, size_t bytes);
  float *getf(const std::string &name, size_t n) { return (float *)get(name, n * sizeof(float)); }
  void *pinned_get(size_t bytes);
  void launched(int n = 1) { launches += n; }
};

// ---------------------------------------------------------------------------
// graph (device CSR lists + per-structure data)
// ---------------------------------------------------------------------------
struct chg_graph {
  chg_ctx *ctx = nullptr;
  uint64_t id = 0;
  int S = 0;
  int64_t N = 0, E = 0, B = 0, A = 0;
  double r_atom = 5.0, r_bond = 3.0;   // model cutoffs (bases and envelopes)
  // fixed-topology (Verlet skin) graphs for captured MD steps: lists built with r + skin,
  // geometry refreshed from new positions by graph_refresh (pos0: positions at the build,
  // geo_dev: the per-structure lattice / inverse table of the build)
  double skin = 0.0;
  double *pos0 = nullptr;
  void *geo_dev = nullptr;
  std::vector<int64_t> atom_ptr_h;     // [S+1]
  std::vector<int64_t> counts_h;       // [S*4] N,E,B,A (filled on demand: graph_fill_counts)
  bool counts_ready = false;
  int *d_flag = nullptr;               // device flags of the build (bit 3: reverse edge missing)
  void *block = nullptr;               // one allocation for all arrays below
  // per atom
  int32_t *atom_ptr = nullptr;         // [S+1]
  int32_t *struct_of_atom = nullptr;   // [N]
  int32_t *species = nullptr;          // [N]
  int32_t *row_ptr = nullptr;          // [N+1] edges by centre
  int32_t *bond_ptr = nullptr;         // [N+1] bonds by centre
  int32_t *atom_angle_ptr = nullptr;   // [N+1] angles by centre
  // per edge
  int32_t *center = nullptr;           // [E]
  int32_t *nbr = nullptr;              // [E]
  char4 *img = nullptr;                // [E] (n1,n2,n3,0)
  float4 *vec = nullptr;               // [E] (dx,dy,dz,|d|) fp32
  double4 *vec64 = nullptr;            // [E] (dx,dy,dz,|d|) fp64 (basis geometry)
  int32_t *bond_id = nullptr;          // [E] or -1
  int32_t *rev = nullptr;              // [E]
  // per bond
  int32_t *bond_edge = nullptr;        // [B]
  int32_t *bond_ctr = nullptr;         // [B] centre atom of the bond
  int32_t *angle_ptr = nullptr;        // [B+1]
  // per angle
  int32_t *angle_b1 = nullptr;         // [A]
  int32_t *angle_b2 = nullptr;         // [A]
  int32_t *angle_e1 = nullptr;         // [A] edge of b1
  int32_t *angle_e2 = nullptr;         // [A] edge of b2
  int32_t *angle_ctr = nullptr;        // [A] centre atom
  int32_t *swap = nullptr;             // [A]
  // per structure
  float *lattice_f = nullptr;          // [S*9]
  float *inv_natoms = nullptr;         // [S]
  // built on ctx's stream; another context of the same device may use it (graph prefetch):
  // its stream waits on `ready`, and the arrays are freed only after that user's work
  cudaEvent_t ready = nullptr;
  chg_ctx *user = nullptr;
};

// ---------------------------------------------------------------------------
// model
// ---------------------------------------------------------------------------
struct chg_model {
  chg_ctx *ctx = nullptr;
  chg_model_cfg cfg{};
  int64_t P = 0;
  float *params = nullptr, *grads = nullptr, *m = nullptr, *v = nullptr;
  std::vector<std::string> names;
  std::vector<const char *> name_ptrs;
  std::vector<int64_t> offsets;
  std::vector<int32_t> shapes;   // 2 per tensor
  std::map<std::string, int> index;
  // table of 2-D tensors for the transposed-weight copy used by the backward
  int n2d = 0;
  int64_t *d_toff = nullptr;
  int32_t *d_trc = nullptr;
  void *tc_cache = nullptr;      // tensor-core weight images per call site (tc_gemm.cu)
  float *wt = nullptr;           // transposed copy of every 2-D weight (same flat offsets)

  int64_t off(const std::string &n) const {
    auto it = index.find(n);
    if (it == index.end()) CHG_THROW(CHG_ERR_ARG, "no parameter %s", n.c_str());
    return offsets[it->second];
  }
  float *p(const std::string &n) const { return params + off(n); }
  float *g(const std::string &n) const { return grads + off(n); }
};

// ---------------------------------------------------------------------------
// device helpers
// ---------------------------------------------------------------------------
// round-to-nearest TF32 (10-bit mantissa) kept in an fp32 container: operands written in this
// form are consumed by the tcgen05 kind::tf32 GEMMs without a conversion pass
__device__ __forceinline__ float tf32_round(float x) {   // = cvt.rna.tf32.f32 (ties away from zero)
  return __uint_as_float((__float_as_uint(x) + 0x1000u) & 0xffffe000u);
}
// SiLU with the approximate reciprocal, as the tensor-core operand paths apply it
__device__ __forceinline__ float silu_fast(float x) { return __fdividef(x, 1.0f + __expf(-x)); }
__device__ __forceinline__ float sigmoidf_(float x) { return 1.0f / (1.0f + __expf(-x)); }
__device__ __forceinline__ float siluf_(float x) { return x * sigmoidf_(x); }
__device__ __forceinline__ float dsiluf_(float x) {
  float s = sigmoidf_(x);
  return s * (1.0f + x * (1.0f - s));
}
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// RAII device-time scope: records an event pair around the launches it covers
// when profiling is on (algorithmic flops / bytes supplied by the caller).
// stable copy of a composed profile tag (ProfScope keeps the pointer)
inline const char *prof_tag(const std::string &t) {
  static std::map<std::string, std::string> pool;
  auto it = pool.emplace(t, t).first;
  return it->second.c_str();
}

struct ProfScope {
  chg_ctx *ctx;
  int ev = -1;
  ProfScope(chg_ctx *c, const char *tag, double flops, double bytes) : ctx(c) {
    if (!ctx->prof_on) return;
    cudaEvent_t a = ctx->next_event();
    ctx->next_event();
    ev = (int)ctx->ev_used - 2;
    cudaEventRecord(a, ctx->stream);
    ctx->prof.push_back({tag, ev, flops, bytes});
  }
  ~ProfScope() {
    if (ev >= 0) cudaEventRecord(ctx->ev_pool[ev + 1], ctx->stream);
  }
};

inline int ceil_div(int64_t a, int64_t b) { return (int)((a + b - 1) / b); }
inline void check_launch(chg_ctx *ctx, const char *file = __builtin_FILE(), int line = __builtin_LINE()) {
  ctx->launched();
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) CHG_THROW(CHG_ERR_CUDA, "kernel launch at %s:%d: %s", file, line, cudaGetErrorString(e));
  static const bool sync_each = getenv("CHG_SYNC_CHECK") != nullptr;   // debug: attribute async faults to a launch
  if (sync_each) {
    e = cudaStreamSynchronize(ctx->stream);
    if (e != cudaSuccess) CHG_THROW(CHG_ERR_CUDA, "kernel at %s:%d: %s", file, line, cudaGetErrorString(e));
  }
}

// Programmatic dependent launch: every kernel is launched with the PDL attribute and starts
// with pdl_begin() — it waits for the preceding kernel of the stream (completion + memory
// flush) and lets the next kernel's CTAs be scheduled as soon as its own CTAs are resident, so
// launch processing and CTA ramp overlap the predecessor's tail.  Nothing is read before the
// wait, so the ordering of the stream is unchanged (CHG_NO_PDL=1: plain launches).  The
// attribute is dropped while a side-stream branch is in flight (ctx->forked).
__device__ __forceinline__ void pdl_begin() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
template <typename... KArgs, typename... Args>
inline void launch_k(chg_ctx *ctx, void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                     Args &&...args) {
  static const bool no_pdl = getenv("CHG_NO_PDL") != nullptr;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  // not while two streams run: early-launched CTAs waiting on their predecessor would hold SM
  // slots the other stream's kernels need (measured: fp32 C2 -12 %, C3 -1 %)
  // (and not inside a stream capture on a multi-rank ctx: the launch failed there, "invalid device
  // function", on NCCL-initialised contexts)
  at[0].val.programmaticStreamSerializationAllowed = (no_pdl || ctx->forked || (ctx->capturing && ctx->nranks > 1)) ? 0 : 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);   // errors: check_launch (cudaGetLastError)
}

// per-device facts and opt-ins (abi.cu): thread-safe, cached per CUDA device, so one process
// may run ctxs on several GPUs (the attribute is per device context)
int device_sm_count();                                  // SMs of the current device
void smem_optin(const void *func, int bytes);           // MaxDynamicSharedMemorySize once per (func, device)

// model.cu: the step's phases (also used by the captured step, capture.cu)
void forward_impl(chg_ctx *ctx, chg_model *m, chg_graph *g, int train, chg_pred *out);
void backward_impl(chg_ctx *ctx, chg_model *m, chg_graph *g, const chg_labels *lab, const chg_loss_cfg *cfg,
                   double *loss_out);
void step_impl(chg_ctx *ctx, chg_model *m, const chg_adam_cfg *cfg, int flag_slot /* -1: next free */);
void check_pending(chg_ctx *ctx, bool block);       // deferred finite checks (CHG_ERR_NONFINITE)
// graph.cu: recompute every edge's geometry of a skin graph from positions (device); flag
// (device int32, may be null) <- 1 when an atom moved more than skin / 2 since the build
void graph_refresh(chg_ctx *ctx, chg_graph *g, const double *pos, int32_t *flag);
void push_pending(chg_ctx *ctx, int slot, const chg_model *m);
int next_flag_slot(chg_ctx *ctx);

// reduce.cu
float *red_partial(chg_ctx *ctx, size_t floats);       // partial buffer for the next recorded job
void red_push(chg_ctx *ctx, RedJob j);                 // record (red_on) or launch now
void red_flush(chg_ctx *ctx);                          // one launch for every recorded job

// graph.cu
chg_graph *build_graph_impl(chg_ctx *ctx, int S, const int64_t *atom_ptr, const double *pos,
                            const double *lat, const int32_t *species, double r_atom, double r_bond,
                            int on_device, int n_species, double skin = 0.0);
