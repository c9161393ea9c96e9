/* chg.h — C ABI of libchg: the FastCHGNet training step on B200 (sm_100a).
 *
 * Method: arXiv 2412.20796.  Every entry point cites the passage
 * that defines its operation.  Readings of ambiguous passages: DESIGN.md.
 *
 * Conventions (all calls):
 *   - Row-vector convention: lattice rows are the lattice vectors a1,a2,a3 (Å);
 *     linear maps are y = x W + b with W stored [in, out] row-major.
 *   - Every call returns chg_status (0 = CHG_OK).  On failure the call has no
 *     visible side effects and chg_last_error(ctx) holds one line of detail.
 *   - Host pointers are read only during the call (the library copies them).
 *     Device pointers (flag `*_on_device` = 1) must stay valid until the work
 *     enqueued on the ctx stream has finished.
 *   - Handles are owned by the caller and released with the *_destroy calls.
 *     A model is bound to the ctx (device) that created it.  A graph may be
 *     used by another ctx of the same device (graph prefetch: a builder ctx
 *     builds batch i+1 on its own stream while the training ctx runs batch i):
 *     the using ctx's stream waits for the build, and chg_graph_destroy
 *     releases the arrays only after the user's enqueued work (one user ctx
 *     per graph besides its builder; CHG_ERR_ARG otherwise).
 *   - A ctx is not thread-safe; use one per (thread, device).
 *   - Determinism: same inputs -> bit-identical outputs, gradients and
 *     parameters on a given GPU count (no atomics on the feature path, fixed
 *     reduction trees).
 */
#ifndef CHG_H_
#define CHG_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  CHG_OK = 0,
  CHG_ERR_ARG = 1,        /* bad argument (null pointer, size, config)            */
  CHG_ERR_GEOMETRY = 2,   /* |det L| <= 1e-6 Å^3, non-finite input, coincident atoms */
  CHG_ERR_SPECIES = 3,    /* Z outside 1..n_species                               */
  CHG_ERR_CAPACITY = 4,   /* a count does not fit the int32 index space           */
  CHG_ERR_NONFINITE = 5,  /* non-finite gradient found by chg_step                */
  CHG_ERR_CUDA = 6,       /* CUDA runtime error (message has the CUDA string)     */
  CHG_ERR_NCCL = 7,       /* NCCL error                                           */
  CHG_ERR_STATE = 8       /* call order violated (e.g. backward without forward)  */
} chg_status;

typedef struct chg_ctx chg_ctx;      /* device, stream, workspaces, optional NCCL communicator */
typedef struct chg_graph chg_graph;  /* device CSR batch graph (atom graph, bond graph, angles) */
typedef struct chg_model chg_model;  /* flat fp32 params | grads | Adam m | Adam v + layout    */

/* Cutoffs of the atom graph and the bond graph (NS: 5 Å / 3 Å).
 * Require 0 < r_bond <= r_atom. */
typedef struct { double r_atom, r_bond; } chg_cutoffs;

/* Model hyper-parameters (d = 64, 31 radial / 31 angular bases, p = 8).
 * n_atom_conv = 4 and n_bond_conv = 3: three interaction blocks (Eq. 3,
 * t = 0,1,2) plus a final atom conv; the angle update of the last block has no
 * consumer and is skipped (reading Q17).  gmlp_hidden = 64: each
 * GatedMLP branch of atom/bond conv is Linear-SiLU-Linear (reading Q12).
 * mlp_precision (the GatedMLP contractions; everything else is fp32 on CUDA cores):
 *   0 = fp32 CUDA cores (strict parity: gradients <= 1e-4);
 *   1 = 3xTF32 on the tcgen05 tensor cores: each operand split x = hi + lo (both TF32)
 *       and A_lo·B_hi + A_hi·B_lo + A_hi·B_hi accumulated in fp32 (fp32-level accuracy,
 *       the strict 1e-4 gradient bar; the paper trains in fp32);
 *   2 = TF32 on the tcgen05 tensor cores (gradients <= 2e-3, NS "loosened" mode);
 *   3 = BF16 on the tcgen05 tensor cores (kind::f16, fp32 accumulate): GEMM operands are
 *       rounded to BF16 as they are staged, features stay fp32 in HBM (the NS 2e-3
 *       gradient bar; a weight gradient with indexed D rows runs in TF32).
 * Any other value is CHG_ERR_ARG at chg_model_create.  Only d = 64, n_radial = n_angular = 31, gmlp_hidden = head_hidden = 64 are built. */
typedef struct {
  int d, n_radial, n_angular, envelope_p, n_atom_conv, n_bond_conv, gmlp_hidden,
      n_species, head_hidden, mlp_precision;
} chg_model_cfg;

/* Outputs of chg_forward (Fig. 1a: E, F, σ, m).  Sizes S, N from the graph.
 * energy [S] eV, energy_per_atom [S] eV/atom, forces [N*3] eV/Å,
 * stress [S*9] GPa (row-major 3x3), magmom [N] μB.  NULL field = not copied.
 * on_device = 1: pointers are device memory (written asynchronously). */
typedef struct {
  float *energy, *energy_per_atom, *forces, *stress, *magmom;
  int on_device;
} chg_pred;

/* Labels for the loss.  energy_per_atom [S], forces [N*3],
 * stress [S*9], magmom [N], magmom_mask [N] (1 = labelled).  A NULL array
 * skips that task (its loss term and seeds are 0); a NULL
 * magmom_mask with magmom given means every atom is labelled.  All four
 * label arrays NULL is CHG_ERR_ARG (chg_backward). */
typedef struct {
  const float *energy_per_atom, *forces, *stress, *magmom;
  const uint8_t *magmom_mask;
  int on_device;
} chg_labels;

/* Huber multi-task loss (prefactors 2, 1.5, 0.1, 0.1; δ reading Q22).
 * The normalisers are GLOBAL counts over all ranks (structures, atoms,
 * labelled magmoms) so that per-rank gradients add up to the full-batch
 * gradient (reading Q23).  A count <= 0 means "this batch's count". */
typedef struct {
  float w_e, w_f, w_s, w_m, huber_delta;
  int64_t n_struct_global, n_atoms_global, n_magmom_global;
} chg_loss_cfg;

/* Adam (PyTorch semantics, no weight decay).  `step` is the 1-based
 * step number used for bias correction.  lr comes from Eq. 14 × cosine
 * (computed by the caller).  allreduce = 1: sum gradients over the NCCL
 * communicator set with chg_ctx_set_nccl before the update.
 * defer_check = 1: no host synchronisation in chg_step — the update is still
 * skipped ON THE DEVICE when a gradient is non-finite, and CHG_ERR_NONFINITE
 * (naming the tensor) is returned by a later chg_step / chg_exec_step /
 * chg_sync on the ctx once the flag's copy has completed. */
typedef struct {
  float lr, beta1, beta2, eps;
  int64_t step;
  int allreduce;
  int defer_check;
} chg_adam_cfg;

/* ---- context ------------------------------------------------------------ */
/* device: CUDA ordinal.  cuda_stream: a cudaStream_t to enqueue on, or NULL
 * for a stream owned by the ctx. */
chg_status chg_ctx_create(int device, void *cuda_stream, chg_ctx **out);
void chg_ctx_destroy(chg_ctx *ctx);
/* One line describing the last failure on ctx (valid until the next call). */
const char *chg_last_error(const chg_ctx *ctx);
/* Waits for the ctx stream; surfaces asynchronous CUDA errors. */
chg_status chg_sync(chg_ctx *ctx);
/* Number of kernels this ctx has launched so far (bench/tests bookkeeping). */
int64_t chg_launch_count(const chg_ctx *ctx);

/* NCCL bootstrap for data parallelism.  uid: 128 bytes from
 * chg_nccl_unique_id on rank 0, broadcast by the caller. */
chg_status chg_nccl_unique_id(void *uid128);
chg_status chg_ctx_set_nccl(chg_ctx *ctx, const void *uid128, int nranks, int rank);
/* SURVEY §8(f) NEXT-3 ("perform all-reduce once after the gradient calculation of a
 * part of parameters is completed"): on = 1 makes every chg_backward on a multi-rank ctx sum
 * the gradients over the ranks in buckets while it runs — the heads + last atom conv, then
 * each (atom, bond, angle) layer, then embedding / bases — one grouped ncclAllReduce per
 * bucket on a communication stream, overlapping the backward of the earlier layers; the
 * following chg_step only waits for them (its own allreduce is skipped).  Exactly one
 * chg_backward per chg_step while on (a second one would add to already-summed gradients). */
chg_status chg_ctx_set_grad_overlap(chg_ctx *ctx, int on);

/* ---- A1 graph build (Alg. 2; reading Q8-Q11) ------------
 * Builds, for S structures, the atom graph (all (i, j, n) with
 * |r_i - (r_j + n L)| <= r_atom, self-image n = 0 excluded), the bond flags
 * (<= r_bond), the ordered angle pairs of distinct bond edges sharing a
 * centre, the reverse-edge map and the angle swap map.  Lists are CSR-sorted
 * by centre atom and match the fp64 oracle bit-exactly (canonical fp64
 * evaluation, reading Q10).
 *   atom_ptr  [S+1] int64 (host memory always)
 *   positions [N*3] fp64 Cartesian Å (not wrapped)
 *   lattice   [S*9] fp64 rows = lattice vectors
 *   species   [N]   int32 Z in 1..94
 *   inputs_on_device: 1 = positions/lattice/species are device pointers.
 * Errors: CHG_ERR_ARG, CHG_ERR_GEOMETRY, CHG_ERR_SPECIES, CHG_ERR_CAPACITY. */
chg_status chg_build_graph(chg_ctx *ctx, int32_t n_struct, const int64_t *atom_ptr,
                           const double *positions, const double *lattice,
                           const int32_t *species, chg_cutoffs cutoffs,
                           int inputs_on_device, chg_graph **out);
/* tot = {N, E, B, A}; per_struct (optional, host) = S rows of {N_s, E_s, B_s, A_s}. */
chg_status chg_graph_counts(const chg_graph *g, int64_t tot[4], int64_t *per_struct);
/* Copies the graph lists to caller-allocated HOST arrays (sizes from counts):
 * row_ptr [N+1], nbr [E], img [E*3] int8, vec [E*4] fp32 (dx,dy,dz,|d|),
 * bond_id [E], bond_edge [B], angle_ptr [B+1], angle_b1 [A], angle_b2 [A],
 * rev [E], swap [A].  Any pointer may be NULL (skipped). Synchronises. */
chg_status chg_graph_export(const chg_graph *g, int32_t *row_ptr, int32_t *nbr, int8_t *img,
                            float *vec, int32_t *bond_id, int32_t *bond_edge,
                            int32_t *angle_ptr, int32_t *angle_b1, int32_t *angle_b2,
                            int32_t *rev, int32_t *swap);
void chg_graph_destroy(chg_graph *g);
/* Make ctx's stream wait for the build of g (built by ctx or by another ctx of the same
 * device — graph prefetch, see the conventions above); chg_forward does this implicitly.
 * Registers ctx as the graph's user.  CHG_ERR_ARG for another device or a third ctx. */
chg_status chg_graph_wait(chg_ctx *ctx, chg_graph *g);

/* ---- model ------------------------------------------------------------- */
chg_status chg_model_create(chg_ctx *ctx, const chg_model_cfg *cfg, chg_model **out);
void chg_model_destroy(chg_model *m);
/* Canonical flat layout: n tensors, names,
 * offsets into the flat vector, shapes (n x 2; 1-D tensors have shape[1] = 0).
 * Arrays are owned by the model. */
chg_status chg_model_layout(const chg_model *m, int *n, const char *const **names,
                            const int64_t **offsets, const int32_t **shapes);
int64_t chg_model_num_params(const chg_model *m);
/* Host <-> device copies of the flat fp32 vectors (n must equal num_params).
 * which: 0 = params, 1 = grads, 2 = Adam m, 3 = Adam v. */
chg_status chg_model_set(chg_model *m, int which, const float *host, int64_t n);
chg_status chg_model_get(const chg_model *m, int which, float *host, int64_t n);
/* Device pointer of a flat vector (which as above), for collectives. */
void *chg_model_device_ptr(chg_model *m, int which);

/* ---- A2-A6 forward (Eq. 2-9 with Eq. 11; Fig. 2a) -----------------------
 * train = 1 keeps the activations needed by chg_backward in the ctx
 * workspace (valid until the next chg_forward on ctx). */
chg_status chg_forward(chg_ctx *ctx, chg_model *m, chg_graph *g, int train, chg_pred *out);

/* ---- conservative forces (the reference-CHGNet output) --
 * Same outputs as chg_forward except forces and stress, which are the derivatives of the
 * energy head instead of the decomposed heads (Eq. 7 / Eq. 9):
 *   forces[i] = −∂E/∂r_i (eV/Å),  stress[s] = (160.21766208 / V_s)·∂E_s/∂ε_s (GPa, reading Q27,
 *   r → r(I+ε), L → L(I+ε), graph fixed); energy, energy_per_atom, magmom as in chg_forward.
 * One forward pass plus a first-order backward seeded with ∂E/∂e_atom = 1 (parameter
 * gradients untouched) and analytic basis derivatives (fp64 geometry).  Consumes the
 * train-mode activations: a following chg_backward needs a new chg_forward (CHG_ERR_STATE). */
chg_status chg_forward_conservative(chg_ctx *ctx, chg_model *m, chg_graph *g, chg_pred *out);

/* ---- MD inference loop (Table II regime) ----------------
 * One half of a velocity-Verlet NVE step on device arrays (all DEVICE pointers, enqueued on
 * the ctx stream; units eV, Å, amu, fs):
 *   drift = 1:  v += (dt/2)·F/m·c, then r += dt·v     (call before rebuilding the graph)
 *   drift = 0:  v += (dt/2)·F/m·c                     (call with the new forces)
 * c = 9.648533212e-3 Å/fs² per eV/(Å·amu).  positions / velocities: fp64 [n,3]; forces: fp32
 * [n,3] (e.g. chg_forward_conservative with on_device outputs); inv_mass: fp64 [n] (1/amu).
 * Periodic wrapping is not applied (the graph builder accepts any Cartesian positions).
 * Errors: CHG_ERR_ARG for null pointers with n > 0. */
chg_status chg_md_verlet(chg_ctx *ctx, int64_t n_atoms, double *positions, double *velocities, const float *forces,
                         const double *inv_mass, double dt_fs, int drift);

/* Fixed-topology (Verlet skin) graphs, so that an MD step has constant sizes and can be
 * captured.  chg_build_graph_skin builds the lists of chg_build_graph with the LIST cutoffs
 * r_atom + skin and r_bond + skin while the model keeps r_atom / r_bond: the radial bases
 * and their envelope u(r / r_c) are exactly zero for r >= r_c (u(1) = u'(1) = u''(1) = 0,
 * reading Q2), so the extra pairs carry zero messages (Eq. 4 / 5 are products with eᵃ, eᵇ) and
 * the energy and conservative forces equal those of the exact lists (summation order aside)
 * for as long as no atom has moved more than skin / 2 since the build.  Same arguments and
 * errors as chg_build_graph plus 0 <= skin < r_atom (CHG_ERR_ARG).
 * chg_graph_refresh recomputes every edge's geometry of such a graph from new positions
 * (DEVICE fp64 [N*3], same atom order) by the build's canonical fp64 evaluation; the lists,
 * bond flags and angles stay those of the build.  flag (DEVICE int32, may be NULL) is set to 1
 * — never cleared — when an atom moved more than skin / 2 since the build: rebuild then.
 * Enqueued on the ctx stream, no host synchronisation. */
chg_status chg_build_graph_skin(chg_ctx *ctx, int32_t n_struct, const int64_t *atom_ptr,
                                const double *positions, const double *lattice,
                                const int32_t *species, chg_cutoffs cutoffs, double skin,
                                int inputs_on_device, chg_graph **out);
chg_status chg_graph_refresh(chg_ctx *ctx, chg_graph *g, const double *positions, int32_t *flag);

/* Captured MD step: chg_md_capture records one velocity-Verlet step on a
 * skin graph — kick + drift (chg_md_verlet drift = 1), chg_graph_refresh(positions, flag),
 * chg_forward_conservative into out (DEVICE pointers, on_device = 1; out->forces required) and
 * the closing kick — as one CUDA graph; it first runs chg_forward_conservative once (sizing the
 * workspaces; out then holds the forces of the current positions, as the first kick needs).
 * chg_md_run replays it n_steps times on the ctx stream (no host work per step).  All
 * pointers must stay valid while the exec is used; it is bound to (ctx, model, g) and becomes
 * invalid (CHG_ERR_STATE) when a ctx workspace was re-allocated after the capture.  The caller
 * checks flag between runs (it only grows) and rebuilds the graph and the exec when it is set. */
typedef struct chg_md_exec chg_md_exec;
chg_status chg_md_capture(chg_ctx *ctx, chg_model *m, chg_graph *g, double *positions, double *velocities,
                          const double *inv_mass, double dt_fs, const chg_pred *out, int32_t *flag,
                          chg_md_exec **exec);
chg_status chg_md_run(chg_ctx *ctx, chg_md_exec *x, int n_steps);
void chg_md_exec_destroy(chg_md_exec *x);

/* ---- A7-A8 loss + backward (first-order only) ---------
 * Computes the Huber loss of the last train-mode forward and ACCUMULATES
 * dL/dθ into the model's gradient vector.  loss_out (host, optional) =
 * {total, E, F, S, M}; NULL = no host synchronisation.
 * Errors: CHG_ERR_STATE if the last forward on ctx was not train-mode on g;
 * CHG_ERR_ARG if every label array is NULL. */
chg_status chg_backward(chg_ctx *ctx, chg_model *m, chg_graph *g, const chg_labels *labels,
                        const chg_loss_cfg *cfg, double loss_out[5]);

/* ---- A9 allreduce + Adam ---------------------------------
 * [ncclAllReduce(sum) of the gradients if cfg->allreduce] -> finite check ->
 * Adam update of params/m/v -> gradients zeroed.  On a non-finite gradient
 * returns CHG_ERR_NONFINITE naming the first offending tensor and leaves
 * params, m and v untouched (gradients are kept — with allreduce they already
 * hold the cross-rank sum, so every rank sees the same non-finite entry and
 * takes the same decision; do not reduce them again).  Synchronises once (the
 * finite flag). */
chg_status chg_step(chg_ctx *ctx, chg_model *m, const chg_adam_cfg *cfg);

/* ---- captured training step (CUDA graph) ----------
 * chg_capture_step records forward(train) + backward + [allreduce] + finite
 * check + Adam on graph g into one CUDA graph (no host synchronisation inside):
 * it first runs forward + backward once on the stream (sizing every workspace;
 * the gradients are restored afterwards), then captures.  labels must be
 * DEVICE pointers (on_device = 1) that stay valid while the exec is used;
 * adam->defer_check is implied.  chg_exec_step replays it with this step's lr
 * and bias-correction step (the Adam node's scalars are updated in the
 * instantiated graph), enqueued on the ctx stream; a non-finite gradient is
 * reported by a later call (see defer_check).  The exec is bound to (ctx,
 * model, g); it becomes invalid (CHG_ERR_STATE) when any ctx workspace was
 * re-allocated after the capture (e.g. a larger batch ran: capture after the
 * largest one) and must not outlive g.
 * Errors: CHG_ERR_ARG (host labels), CHG_ERR_STATE, CHG_ERR_CUDA. */
typedef struct chg_exec chg_exec;
chg_status chg_capture_step(chg_ctx *ctx, chg_model *m, chg_graph *g, const chg_labels *labels,
                            const chg_loss_cfg *loss, const chg_adam_cfg *adam, chg_exec **out);
chg_status chg_exec_step(chg_ctx *ctx, chg_exec *x, const chg_adam_cfg *adam);
void chg_exec_destroy(chg_exec *x);

/* ---- load-balance sampler (Fig. 4) -- host only --------------
 * loads[n] = atoms + bonds + angles per sample.  Sort ascending (ties
 * by index); ranks take turns round-robin, each turn taking the smallest and
 * the largest remaining sample.  rank_of[n] (out) = rank of each sample.
 * Errors: CHG_ERR_ARG if n_ranks <= 0 or n < 0. */
chg_status chg_balance(const int64_t *loads, int32_t n, int32_t n_ranks, int32_t *rank_of);

/* ---- measurement -----------------------------------------------------------
 * chg_profile(ctx, 1) clears and enables per-op device timing (CUDA events on
 * the ctx stream around each op group); 0 clears and disables.
 * chg_profile_query(ctx, idx, ...) synchronises and returns, for the idx-th op
 * tag seen since enabling: tag (char[64]), total device ms, number of scopes,
 * and the algorithmic flops / bytes those scopes declared (DESIGN.md
 * "Algorithmic bytes").  CHG_ERR_ARG when idx is past the last tag. */
chg_status chg_profile(chg_ctx *ctx, int mode);
chg_status chg_profile_query(chg_ctx *ctx, int idx, char *tag, double *ms, int64_t *launches, double *flops,
                             double *bytes);

/* ---- kernel unit tests ---------------------------------------------------------
 * chg_debug_gemm runs one GEMM engine on dense host matrices (row-major fp32):
 *   kind 0: out[M,N] = A[M,K] · W[K,N]          (row GEMM; W is also given K-major
 *           internally for the tensor-core path)
 *   kind 1: out[K,N] = A[M,K]ᵀ · D[M,N]         (weight-gradient GEMM; `W` = D)
 * engine 0 = fp32 CUDA cores, 1 = tcgen05 3xTF32, 2 = tcgen05 TF32, 3 = tcgen05 BF16.  Returns CHG_ERR_ARG if the
 * engine cannot run the shape.  Synchronises. */
chg_status chg_debug_gemm(chg_ctx *ctx, int kind, int engine, int M, int K, int N, const float *A,
                          const float *W, float *out);

/* ---- debugging / parity ---------------------------------------------------
 * Copies a named intermediate of the last forward/backward to host memory:
 * names "ea_t","eb_t","a_t" (bases, [rows,32] zero-padded), "v0".."v4",
 * "e0".."e3","ea","eb","a0".."a2".  n = capacity in floats; *rows/*cols out. */
chg_status chg_debug_get(chg_ctx *ctx, const char *name, float *host, int64_t n, int64_t *rows,
                         int64_t *cols);

#ifdef __cplusplus
}
#endif
#endif /* CHG_H_ */
