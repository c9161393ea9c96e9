// md.cu — velocity-Verlet NVE integrator of the MD inference loop.
//
// The forces come from chg_forward_conservative (F = −∂E/∂r of the energy head); the graph is
// rebuilt every step by chg_build_graph from the device-resident positions (cell lists for
// large cells).  One step of velocity Verlet (units eV, Å, amu, fs):
//   drift = 1:  v ← v + (dt/2)·a(t),  r ← r + dt·v          (before the new forces)
//   drift = 0:  v ← v + (dt/2)·a(t+dt)                       (after them)
// with a = F / m · 9.648533212e-3 Å/fs² per eV/(Å·amu).  fp64 state, fp32 forces.
#include "common.cuh"

namespace {

constexpr double ACC_UNIT = 9.648533212e-3;   // (eV/Å)/amu -> Å/fs²

__global__ void k_verlet(int64_t n, double *__restrict__ pos, double *__restrict__ vel, const float *__restrict__ F,
                         const double *__restrict__ inv_mass, double dt, int drift) {
  pdl_begin();
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double h = 0.5 * dt * ACC_UNIT * inv_mass[i];
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    const double v = vel[3 * i + c] + h * (double)F[3 * i + c];
    vel[3 * i + c] = v;
    if (drift) pos[3 * i + c] += dt * v;
  }
}

}  // namespace

void md_verlet(chg_ctx *ctx, int64_t n, double *pos, double *vel, const float *F, const double *inv_mass, double dt,
               int drift) {
  if (n <= 0) return;
  ProfScope ps(ctx, "md_verlet", 0.0, n * (drift ? 68.0 : 44.0));
  launch_k(ctx, k_verlet, ceil_div(n, 256), 256, 0, ctx->stream, n, pos, vel, F, inv_mass, dt, drift);
  check_launch(ctx);
}
