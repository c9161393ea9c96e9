// deriv.cu — conservative forces and stress of the energy head (the
// reference-CHGNet output: P:141; reading Q27 for the stress convention):
//   F_i = −∂E/∂r_i,   σ_s = (160.21766208 / V_s) · ∂E_s/∂ε_s   (graph fixed, r → r(I+ε), L → L(I+ε)).
//
// E depends on the positions only through the edge vectors d_e = r_i − (r_j + n L) (the
// radial bases of the atom and bond graphs and the angle Fourier basis), so with
// g_e = ∂E/∂d_e:  F_i = −Σ_{e out of i} (g_e − g_rev(e))  and  ∂E/∂ε = Σ_e d_e ⊗ g_e.
// g_e is assembled from the backward's dE/d(e⁰, eᵃ, eᵇ, a⁰) (a first-order backward seeded with
// ∂E/∂e_atom = 1, no parameter gradients) through the basis projections and the analytic
// derivatives of the bases (fp64 geometry):
//   radial:  ∂B_n/∂r with B_n = u(r/r_c)·√(2/r_c)·sin(f_n r/r_c)/r  (envelope u of reading Q2)
//   angle:   ∂v_k/∂cosθ for the Fourier features (Q6) and ∂cosθ/∂d of the two bond vectors.
// Every sum has a fixed order (warp trees, CSR rows, swap permutation): deterministic.
#include <cmath>

#include "ops.cuh"

namespace {

__device__ __forceinline__ void envelope_du(double xi, int p, double &u, double &du) {
  if (xi >= 1.0) { u = 0.0; du = 0.0; return; }       // clamped beyond the cutoff (proj.cu)
  double xp1 = 1.0;                                   // xi^(p-1)
  for (int k = 0; k < p - 1; ++k) xp1 *= xi;
  const double xp = xp1 * xi;
  const double a = 0.5 * (p + 1) * (p + 2), b = (double)p * (p + 2), c = 0.5 * p * (p + 1);
  u = 1.0 - xp * (a - xi * (b - c * xi));
  du = -xp1 * (a * p - xi * (b * (p + 1) - c * (p + 2) * xi));
}

__device__ __forceinline__ float warp_sum_f(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// warp per basis row; lane n = basis function.  dE/dB_n = Σ_c dE[c]·W[n][c] over the NC
// projections (W row-major [31][64] each, held transposed in shared memory), then
// Σ_n dE/dB_n · ∂B_n/∂r → g_e (+)= that · d_e / r   (e = eor ? eor[row] : row).
template <int NC>
__global__ void __launch_bounds__(256) k_dgeom_radial(int64_t rows, const double4 *__restrict__ vec,
                                                      const int32_t *__restrict__ eor, const float *__restrict__ freq,
                                                      double rc, int p, const float *__restrict__ W0,
                                                      const float *__restrict__ W1, const float *__restrict__ dE0,
                                                      const float *__restrict__ dE1, float4 *__restrict__ g,
                                                      int accumulate) {
  pdl_begin();
  __shared__ float Wt[NC * 64][33];
  __shared__ float rowbuf[8][NC * 64];
#pragma unroll 8   // independent loads in flight (one latency, not one per iteration)
  for (int i = threadIdx.x; i < NC * 64 * 32; i += blockDim.x) {
    const int c = i / 32, n = i % 32;
    Wt[c][n] = n < CHG_K ? (c < 64 ? W0 : W1)[n * 64 + (c & 63)] : 0.f;
  }
  __syncthreads();
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const double f = lane < CHG_K ? (double)freq[lane] : 0.0;
  const double K = sqrt(2.0 / rc);
  for (int64_t row = blockIdx.x * 8 + w; row < rows; row += (int64_t)gridDim.x * 8) {
#pragma unroll
    for (int q = 0; q < NC * 2; ++q) {
      const int c = lane + 32 * q;
      rowbuf[w][c] = (c < 64 ? dE0 : dE1)[row * 64 + (c & 63)];
    }
    __syncwarp();
    float dEdB = 0.f;
#pragma unroll 8
    for (int c = 0; c < NC * 64; ++c) dEdB = fmaf(rowbuf[w][c], Wt[c][lane], dEdB);
    __syncwarp();
    const int e = eor ? eor[row] : (int)row;
    const double4 d = vec[e];
    const double r = d.w, xi = r / rc;
    double u, du;
    envelope_du(xi, p, u, du);
    double sn, cs;
    sincos(f * xi, &sn, &cs);
    const double dBdr = lane < CHG_K ? K * ((du / rc) * sn / r + u * cs * (f / rc) / r - u * sn / (r * r)) : 0.0;
    const float t = warp_sum_f((float)((double)dEdB * dBdr));
    if (lane == 0) {
      const float sc = (float)((double)t / r);
      float4 v = make_float4(sc * (float)d.x, sc * (float)d.y, sc * (float)d.z, 0.f);
      if (accumulate) { const float4 o = g[e]; v.x += o.x; v.y += o.y; v.z += o.z; }
      g[e] = v;
    }
  }
}

// warp per angle; lane k = Fourier feature.  ∂E/∂cosθ = Σ_k dE/dv_k · ∂v_k/∂cosθ with
// v_{2m-1} = cos(mθ)/√π, v_{2m} = sin(mθ)/√π:  ∂cos(mθ)/∂c = m sin(mθ)/sinθ,
// ∂sin(mθ)/∂c = −m cos(mθ)/sinθ; then the two bond vectors' shares via ∂c/∂d1, ∂c/∂d2.
__global__ void __launch_bounds__(256) k_dgeom_angle(int64_t A, const double4 *__restrict__ vec,
                                                     const int32_t *__restrict__ e1, const int32_t *__restrict__ e2,
                                                     const float *__restrict__ Wth, const float *__restrict__ da,
                                                     float4 *__restrict__ ga1, float4 *__restrict__ ga2) {
  pdl_begin();
  __shared__ float Wt[64][33];
  __shared__ float rowbuf[8][64];
#pragma unroll 8   // independent loads in flight (one latency, not one per iteration)
  for (int i = threadIdx.x; i < 64 * 32; i += blockDim.x) {
    const int c = i / 32, n = i % 32;
    Wt[c][n] = n < CHG_K ? Wth[n * 64 + c] : 0.f;
  }
  __syncthreads();
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const double isp = 0.56418958354775628695;          // 1/√π
  for (int64_t a = blockIdx.x * 8 + w; a < A; a += (int64_t)gridDim.x * 8) {
    rowbuf[w][lane] = da[a * 64 + lane];
    rowbuf[w][lane + 32] = da[a * 64 + lane + 32];
    __syncwarp();
    float dEdv = 0.f;
#pragma unroll 8
    for (int c = 0; c < 64; ++c) dEdv = fmaf(rowbuf[w][c], Wt[c][lane], dEdv);
    __syncwarp();
    const double4 d1 = vec[e1[a]], d2 = vec[e2[a]];
    double c = (d1.x * d2.x + d1.y * d2.y + d1.z * d2.z) / (d1.w * d2.w);
    c = fmin(1.0, fmax(-1.0, c));
    const double sn = fmax(sqrt(fmax(0.0, 1.0 - c * c)), 1e-12);
    const double th = atan2(sn, c);
    double dvdc = 0.0;
    if (lane >= 1 && lane < CHG_K) {
      const int m = (lane + 1) / 2;
      double sm, cm;
      sincos(m * th, &sm, &cm);
      dvdc = (lane & 1) ? m * sm / sn * isp : -m * cm / sn * isp;
    }
    const float G = warp_sum_f((float)((double)dEdv * dvdc));
    if (lane == 0) {
      const double inv12 = 1.0 / (d1.w * d2.w), i11 = 1.0 / (d1.w * d1.w), i22 = 1.0 / (d2.w * d2.w);
      ga1[a] = make_float4((float)(G * (d2.x * inv12 - c * d1.x * i11)), (float)(G * (d2.y * inv12 - c * d1.y * i11)),
                           (float)(G * (d2.z * inv12 - c * d1.z * i11)), 0.f);
      ga2[a] = make_float4((float)(G * (d1.x * inv12 - c * d2.x * i22)), (float)(G * (d1.y * inv12 - c * d2.y * i22)),
                           (float)(G * (d1.z * inv12 - c * d2.z * i22)), 0.f);
    }
  }
}

// edge e with bond b: g_e += Σ_{angles with first bond b} ga1 + Σ_{angles with second bond b} ga2
// (the latter through the swap permutation), in angle order
__global__ void k_angle_to_edge(int64_t E, const int32_t *__restrict__ bond_id, const int32_t *__restrict__ angle_ptr,
                                const int32_t *__restrict__ swp, const float4 *__restrict__ ga1,
                                const float4 *__restrict__ ga2, float4 *__restrict__ g) {
  pdl_begin();
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= E) return;
  const int b = bond_id[e];
  if (b < 0) return;
  float4 acc = g[e];
  for (int a = angle_ptr[b]; a < angle_ptr[b + 1]; ++a) {
    const float4 x = ga1[a], y = ga2[swp[a]];
    acc.x += x.x + y.x; acc.y += x.y + y.y; acc.z += x.z + y.z;
  }
  g[e] = acc;
}

// F_i = −Σ_{e out of i} (g_e − g_rev(e)), warp per atom (fixed tree)
__global__ void k_dforce(int64_t N, const int32_t *__restrict__ row_ptr, const int32_t *__restrict__ rev,
                         const float4 *__restrict__ g, float *__restrict__ F) {
  pdl_begin();
  const int64_t i = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (i >= N) return;
  float fx = 0.f, fy = 0.f, fz = 0.f;
  for (int e = row_ptr[i] + lane; e < row_ptr[i + 1]; e += 32) {
    const float4 a = g[e], b = g[rev[e]];
    fx += a.x - b.x; fy += a.y - b.y; fz += a.z - b.z;
  }
  fx = warp_sum_f(fx); fy = warp_sum_f(fy); fz = warp_sum_f(fz);
  if (lane == 0) { F[3 * i] = -fx; F[3 * i + 1] = -fy; F[3 * i + 2] = -fz; }
}

// σ_s = (160.21766208 / V_s) Σ_{e in s} d_e ⊗ g_e, block per structure (fp64, fixed tree)
__global__ void k_dstress(const int32_t *__restrict__ atom_ptr, const int32_t *__restrict__ row_ptr,
                          const double4 *__restrict__ vec, const float4 *__restrict__ g, const float *__restrict__ lat,
                          float *__restrict__ stress) {
  pdl_begin();
  __shared__ double sh[9][128];
  const int s = blockIdx.x, t = threadIdx.x;
  const int e0 = row_ptr[atom_ptr[s]], e1 = row_ptr[atom_ptr[s + 1]];
  double acc[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
  for (int e = e0 + t; e < e1; e += blockDim.x) {
    const double4 d = vec[e];
    const float4 gg = g[e];
    const double dv[3] = {d.x, d.y, d.z}, gv[3] = {gg.x, gg.y, gg.z};
#pragma unroll
    for (int k = 0; k < 3; ++k)
#pragma unroll
      for (int c = 0; c < 3; ++c) acc[3 * k + c] += dv[k] * gv[c];
  }
#pragma unroll
  for (int q = 0; q < 9; ++q) sh[q][t] = acc[q];
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (t < o)
#pragma unroll
      for (int q = 0; q < 9; ++q) sh[q][t] += sh[q][t + o];
    __syncthreads();
  }
  if (t < 9) {
    const float *l = lat + 9 * s;
    const double det = (double)l[0] * ((double)l[4] * l[8] - (double)l[5] * l[7]) -
                       (double)l[1] * ((double)l[3] * l[8] - (double)l[5] * l[6]) +
                       (double)l[2] * ((double)l[3] * l[7] - (double)l[4] * l[6]);
    stress[9 * s + t] = (float)(160.21766208 * sh[t][0] / fabs(det));
  }
}

__global__ void k_fill_value(int64_t n, float v, float *__restrict__ x) {
  pdl_begin();
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) x[i] = v;
}

int grid_rows(int64_t rows) { return (int)std::max<int64_t>(1, std::min<int64_t>((rows + 7) / 8, 148 * 16)); }

}  // namespace

// geometry part of the conservative-force pass: de, dea, deb, da = dE/d(e⁰, eᵃ, eᵇ, a⁰)
void deriv_geometry(chg_ctx *ctx, const chg_graph *g, const float *freq_a, const float *freq_b, int p,
                    const float *W0, const float *Wa, const float *Wb, const float *Wth, const float *de,
                    const float *dea, const float *deb, const float *da, float *forces, float *stress) {
  const int64_t E = g->E, B = g->B, A = g->A, N = g->N;
  float4 *gv = (float4 *)ctx->get("dgeom_g", 16 * (size_t)std::max<int64_t>(E, 1));
  ProfScope ps(ctx, "deriv_geom", 0.0, E * (512.0 + 48.0) + B * 300.0 + A * 400.0 + N * 12.0);
  if (E > 0) {
    launch_k(ctx, k_dgeom_radial<2>, grid_rows(E), 256, 0, ctx->stream, E, g->vec64, nullptr, freq_a, g->r_atom, p, W0, Wa, de,
                                                             dea, gv, 0);
    check_launch(ctx);
  }
  if (B > 0) {
    launch_k(ctx, k_dgeom_radial<1>, grid_rows(B), 256, 0, ctx->stream, B, g->vec64, g->bond_edge, freq_b, g->r_bond, p, Wb,
                                                             nullptr, deb, nullptr, gv, 1);
    check_launch(ctx);
  }
  if (A > 0) {
    float4 *ga1 = (float4 *)ctx->get("dgeom_a1", 16 * (size_t)A), *ga2 = (float4 *)ctx->get("dgeom_a2", 16 * (size_t)A);
    launch_k(ctx, k_dgeom_angle, grid_rows(A), 256, 0, ctx->stream, A, g->vec64, g->angle_e1, g->angle_e2, Wth, da, ga1, ga2);
    check_launch(ctx);
    launch_k(ctx, k_angle_to_edge, ceil_div(E, 256), 256, 0, ctx->stream, E, g->bond_id, g->angle_ptr, g->swap, ga1, ga2, gv);
    check_launch(ctx);
  }
  if (N > 0) {
    launch_k(ctx, k_dforce, ceil_div(N * 32, 256), 256, 0, ctx->stream, N, g->row_ptr, g->rev, gv, forces);
    check_launch(ctx);
  }
  if (g->S > 0) {
    launch_k(ctx, k_dstress, g->S, 128, 0, ctx->stream, g->atom_ptr, g->row_ptr, g->vec64, gv, g->lattice_f, stress);
    check_launch(ctx);
  }
}

void fill_value(chg_ctx *ctx, float *x, int64_t n, float v) {
  if (n <= 0) return;
  launch_k(ctx, k_fill_value, ceil_div(n, 256), 256, 0, ctx->stream, n, v, x);
  check_launch(ctx);
}
