#include <chrono>
// graph.cu — A1: periodic atom graph, bond graph and angle list on the GPU.
//
// Paper: P:95 (§II-B(1) graph extraction), Alg. 1 lines P:253-256 (r_j += I@L,
// r_ij = r_i − r_j), Alg. 2 P:294-326 (whole batch at once; the block-diagonal
// image matrix is realised per structure segment, never materialised).
// Readings: Q8 directed edges, Q9 ordered angle pairs of distinct
// bond edges, Q10 closed cutoff with ONE canonical fp64 evaluation per
// unordered pair (no FMA: __dmul_rn/__dadd_rn), Q11 d = r_i − (r_j + nL).
//
// Kernels (one warp per centre atom for the pair search, which keeps the
// (i, j, n1, n2, n3) output order without a sort):
//   k_frac      fractional coordinates (image ranges only) + finite/species checks
//   k_count     per centre atom: accepted edges and bond edges          (G1)
//   k_scan      exclusive scans: edges, bonds, angles m(m−1) per atom    (G2)
//   k_fill      ordered emission with warp ballot/scan                  (G3)
//   k_angles    angle pairs, swap map, per-angle edge/centre indices    (G4)
//   k_rev       reverse-edge map by binary search in row j              (G4)
#include <optional>
#include <cmath>

#include "common.cuh"

namespace {

struct StructGeo {
  double L[9];      // rows = lattice vectors
  double Linv[9];
  double rw[3];     // r_atom / perpendicular width
  int nc[3];        // cell-list grid (cells per lattice direction), 0 = brute-force image search
  int pad;
};

// Cell lists for large structures (>= CELL_MIN atoms, every perpendicular width >= 3 cutoffs):
// cells of width >= r_atom, at most one cell per atom (so a structure's cells index into its
// own atom range), 27 neighbour cells per atom.  The accepted pairs are exactly those of the
// brute-force image search (same canonical evaluation of each (i, j, n)); only the candidate
// set shrinks from O(n^2) to O(n).
constexpr int CELL_MIN = 256;
constexpr int CELL_MAXNB = 1024;   // accepted neighbours per atom sorted in shared memory (else brute force)
__host__ __device__ inline void cell_grid(const double rw[3], int64_t n_atoms, int nc[3]) {
  bool ok = n_atoms >= CELL_MIN;
  for (int k = 0; k < 3; ++k) {
    nc[k] = rw[k] > 0 ? (int)floor(1.0 / (rw[k] * (1.0 + 1e-6))) : 0;
    if (nc[k] > 1024) nc[k] = 1024;
    ok = ok && nc[k] >= 3;
  }
  while (ok && (int64_t)nc[0] * nc[1] * nc[2] > n_atoms) {   // larger cells stay valid
    int kmax = 0;
    for (int k = 1; k < 3; ++k)
      if (nc[k] > nc[kmax]) kmax = k;
    if (nc[kmax] <= 3) ok = false;
    else --nc[kmax];
  }
  if (!ok) nc[0] = nc[1] = nc[2] = 0;
}

__device__ __forceinline__ bool lexpos(int n1, int n2, int n3) {
  return n1 > 0 || (n1 == 0 && (n2 > 0 || (n2 == 0 && n3 > 0)));
}

// Canonical evaluation of candidate (i, j, n): see oracle/graph.py docstring.
__device__ __forceinline__ void eval_pair(const double *__restrict__ pos, const double *L, int i, int j,
                                          int n1, int n2, int n3, double &dx, double &dy, double &dz,
                                          double &q) {
  bool flip = (i > j) || (i == j && !lexpos(n1, n2, n3));
  int a = flip ? j : i, b = flip ? i : j;
  double m1 = flip ? -n1 : n1, m2 = flip ? -n2 : n2, m3 = flip ? -n3 : n3;
  double t[3];
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    double v = pos[3 * b + c];
    v = __dadd_rn(v, __dmul_rn(m1, L[0 + c]));
    v = __dadd_rn(v, __dmul_rn(m2, L[3 + c]));
    v = __dadd_rn(v, __dmul_rn(m3, L[6 + c]));
    t[c] = v;
  }
  dx = __dsub_rn(pos[3 * a + 0], t[0]);
  dy = __dsub_rn(pos[3 * a + 1], t[1]);
  dz = __dsub_rn(pos[3 * a + 2], t[2]);
  q = __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
  if (flip) { dx = -dx; dy = -dy; dz = -dz; }
}

struct Range { int lo[3], hi[3]; };

__device__ __forceinline__ Range pair_range(const double *fi, const double *fj, const double *rw) {
  Range r;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    double df = fi[k] - fj[k];
    r.lo[k] = (int)ceil(df - rw[k]) - 1;
    r.hi[k] = (int)floor(df + rw[k]) + 1;
  }
  return r;
}

__global__ void k_frac(int N, const double *__restrict__ pos, const int32_t *__restrict__ soa,
                       const StructGeo *__restrict__ geo, const int32_t *__restrict__ species,
                       int n_species, double *__restrict__ frac, int *flag) {
  pdl_begin();
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= N) return;
  const StructGeo &g = geo[soa[i]];
  double p[3] = {pos[3 * i], pos[3 * i + 1], pos[3 * i + 2]};
  if (!isfinite(p[0]) || !isfinite(p[1]) || !isfinite(p[2])) atomicOr(flag, 1);
  int z = species[i];
  if (z < 1 || z > n_species) atomicOr(flag, 2);
#pragma unroll
  for (int c = 0; c < 3; ++c)
    frac[3 * i + c] = p[0] * g.Linv[0 + c] + p[1] * g.Linv[3 + c] + p[2] * g.Linv[6 + c];
}

// per-structure geometry on the device (inputs already resident: no host round trip).  Same
// formulas as the host path; invalid cells set flag bits 16 / 32 / 64 (non-finite, |det| <= 1e-6,
// too thin) and the smallest offending structure index, and get zero ranges so the later
// kernels stay bounded; the host raises at the size synchronisation.
__global__ void k_geo(int S, const double *__restrict__ lat, double r_atom, const int32_t *__restrict__ atom_ptr,
                      StructGeo *__restrict__ geo, float *__restrict__ lat_f, int *flag) {
  pdl_begin();
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= S) return;
  double l[9];
  bool finite = true;
#pragma unroll
  for (int k = 0; k < 9; ++k) {
    l[k] = lat[9 * s + k];
    finite = finite && isfinite(l[k]);
    lat_f[9 * s + k] = (float)l[k];
  }
  StructGeo g;
  int bad = finite ? 0 : 16;
  const double det = l[0] * (l[4] * l[8] - l[5] * l[7]) - l[1] * (l[3] * l[8] - l[5] * l[6]) +
                     l[2] * (l[3] * l[7] - l[4] * l[6]);
  const double V = fabs(det);
  if (!bad && !(V > 1e-6)) bad = 32;
  const double inv[9] = {l[4] * l[8] - l[5] * l[7], l[2] * l[7] - l[1] * l[8], l[1] * l[5] - l[2] * l[4],
                         l[5] * l[6] - l[3] * l[8], l[0] * l[8] - l[2] * l[6], l[2] * l[3] - l[0] * l[5],
                         l[3] * l[7] - l[4] * l[6], l[1] * l[6] - l[0] * l[7], l[0] * l[4] - l[1] * l[3]};
#pragma unroll
  for (int k = 0; k < 9; ++k) { g.L[k] = l[k]; g.Linv[k] = bad ? 0.0 : inv[k] / det; }
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const double *u = &l[3 * ((k + 1) % 3)], *w = &l[3 * ((k + 2) % 3)];
    const double cx = u[1] * w[2] - u[2] * w[1], cy = u[2] * w[0] - u[0] * w[2], cz = u[0] * w[1] - u[1] * w[0];
    const double width = V / sqrt(cx * cx + cy * cy + cz * cz);
    g.rw[k] = r_atom / width;
    if (!bad && g.rw[k] > 100.0) bad = 64;
  }
  if (bad) {
    for (int k = 0; k < 3; ++k) g.rw[k] = 0.0;
    atomicOr(flag, bad);
    atomicMin(flag + 1, s);
  }
  cell_grid(g.rw, atom_ptr[s + 1] - atom_ptr[s], g.nc);
  g.pad = 0;
  geo[s] = g;
}

__device__ __forceinline__ long long edge_key(int nb, char4 im) {
  return ((long long)nb << 24) | ((long long)((int)im.x + 128) << 16) | ((long long)((int)im.y + 128) << 8) |
         (long long)((int)im.z + 128);
}

// ---- cell lists (structures with g.nc[0] > 0) ----
struct CellArgs {
  int32_t *atom_cell;       // [N] local cell of the atom's wrapped position, -1 = brute-force structure
  int32_t *cell_cnt;        // [N] (structure base + cell) -> atoms; also the placement cursor
  int32_t *cell_start;      // [N + 1]
  int32_t *cell_atoms;      // [N] atoms grouped by cell
};

__device__ __forceinline__ int cell_coord(double f, int nc) {
  const double w = f - floor(f);
  int c = (int)(w * nc);
  return c < 0 ? 0 : (c >= nc ? nc - 1 : c);
}

__global__ void k_cell_assign(int N, const double *__restrict__ frac, const int32_t *__restrict__ soa,
                              const int32_t *__restrict__ atom_ptr, const StructGeo *__restrict__ geo, CellArgs ca) {
  pdl_begin();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= N) return;
  const int s = soa[i];
  const StructGeo &g = geo[s];
  if (g.nc[0] == 0) { ca.atom_cell[i] = -1; return; }
  const int c = (cell_coord(frac[3 * i], g.nc[0]) * g.nc[1] + cell_coord(frac[3 * i + 1], g.nc[1])) * g.nc[2] +
                cell_coord(frac[3 * i + 2], g.nc[2]);
  ca.atom_cell[i] = c;
  atomicAdd(&ca.cell_cnt[atom_ptr[s] + c], 1);
}

// block per structure: exclusive scan of its cell counts -> absolute start positions
__global__ void k_cell_scan(int S, const int32_t *__restrict__ atom_ptr, const StructGeo *__restrict__ geo,
                            CellArgs ca) {
  pdl_begin();
  __shared__ int sh[256];
  const int s = blockIdx.x;
  const StructGeo &g = geo[s];
  if (g.nc[0] == 0) return;
  const int base = atom_ptr[s], ncell = g.nc[0] * g.nc[1] * g.nc[2];
  int carry = base;
  for (int c0 = 0; c0 < ncell; c0 += 256) {
    const int c = c0 + threadIdx.x;
    const int v = c < ncell ? ca.cell_cnt[base + c] : 0;
    sh[threadIdx.x] = v;
    __syncthreads();
    for (int o = 1; o < 256; o <<= 1) {
      const int t = threadIdx.x >= o ? sh[threadIdx.x - o] : 0;
      __syncthreads();
      sh[threadIdx.x] += t;
      __syncthreads();
    }
    if (c < ncell) ca.cell_start[base + c] = carry + sh[threadIdx.x] - v;
    carry += sh[255];
    __syncthreads();
  }
  if (threadIdx.x == 0) ca.cell_start[base + ncell] = carry;   // == atom_ptr[s + 1]
}

__global__ void k_cell_place(int N, const int32_t *__restrict__ soa, const int32_t *__restrict__ atom_ptr,
                             CellArgs ca, int32_t *__restrict__ cursor) {
  pdl_begin();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= N) return;
  const int c = ca.atom_cell[i];
  if (c < 0) return;
  const int base = atom_ptr[soa[i]];
  ca.cell_atoms[ca.cell_start[base + c] + atomicAdd(&cursor[base + c], 1)] = i;
}

// candidate t of atom i's 27 neighbour cells -> (j, n); cnt27 = exclusive prefix of cell sizes
__device__ __forceinline__ void cell_candidate(const CellArgs &ca, int base, const StructGeo &g, int ci0, int ci1,
                                               int ci2, const int *cnt27, int t, const double *frac, const int *si,
                                               int &j, int &n1, int &n2, int &n3) {
  int d = 0;
  while (d < 26 && cnt27[d + 1] <= t) ++d;
  const int dd[3] = {d / 9 - 1, (d / 3) % 3 - 1, d % 3 - 1};
  const int cc[3] = {ci0, ci1, ci2};
  int x[3], w[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    x[k] = cc[k] + dd[k];
    w[k] = 0;
    if (x[k] < 0) { x[k] += g.nc[k]; w[k] = -1; }
    else if (x[k] >= g.nc[k]) { x[k] -= g.nc[k]; w[k] = 1; }
  }
  const int cell = (x[0] * g.nc[1] + x[1]) * g.nc[2] + x[2];
  j = ca.cell_atoms[ca.cell_start[base + cell] + (t - cnt27[d])];
  // d = r_i - (r_j + nL) with wrapped cells: n = shift_i - shift_j + wrap
  n1 = si[0] - (int)floor(frac[3 * j]) + w[0];
  n2 = si[1] - (int)floor(frac[3 * j + 1]) + w[1];
  n3 = si[2] - (int)floor(frac[3 * j + 2]) + w[2];
}

// sizes of atom i's 27 neighbour cells as an exclusive prefix in smem (threads 0..26)
__device__ __forceinline__ void cell_prefix(const CellArgs &ca, int base, const StructGeo &g, int ci, int *cnt27,
                                            int (&cc)[3]) {
  cc[0] = ci / (g.nc[1] * g.nc[2]);
  cc[1] = (ci / g.nc[2]) % g.nc[1];
  cc[2] = ci % g.nc[2];
  if (threadIdx.x < 27) {
    const int d = threadIdx.x;
    const int dd[3] = {d / 9 - 1, (d / 3) % 3 - 1, d % 3 - 1};
    int x[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) x[k] = (cc[k] + dd[k] + g.nc[k]) % g.nc[k];
    const int cell = (x[0] * g.nc[1] + x[1]) * g.nc[2] + x[2];
    cnt27[d + 1] = ca.cell_start[base + cell + 1] - ca.cell_start[base + cell];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    cnt27[0] = 0;
    for (int d = 0; d < 27; ++d) cnt27[d + 1] += cnt27[d];
  }
  __syncthreads();
}

// One 128-thread block (4 warps) per centre atom i.  Lanes walk (j, n1) slots: W >= any pair's
// n1-range width (pair_range: <= 2·rw + 4 values), so a lane runs only the n2 x n3 loops of one
// image row; the four warps take 32-slot chunks round-robin (more warps in flight per SM).
constexpr int GWPA = 4;   // warps per atom

__device__ __forceinline__ int slot_count(const double *__restrict__ pos, const double *__restrict__ frac,
                                          const double *L, const StructGeo &g, const double *fi, int i, int a0,
                                          int W, int p, double ra2, double rb2, int &cb, int &bad, Range &r,
                                          int &j, int &n1) {
  j = a0 + p / W;
  const int k = p % W;
  double fj[3] = {frac[3 * j], frac[3 * j + 1], frac[3 * j + 2]};
  r = pair_range(fi, fj, g.rw);
  n1 = r.lo[0] + k;
  int ce = 0;
  cb = 0;
  if (n1 > r.hi[0]) return 0;
  for (int n2 = r.lo[1]; n2 <= r.hi[1]; ++n2)
    for (int n3 = r.lo[2]; n3 <= r.hi[2]; ++n3) {
      if (i == j && n1 == 0 && n2 == 0 && n3 == 0) continue;
      double dx, dy, dz, q;
      eval_pair(pos, L, i, j, n1, n2, n3, dx, dy, dz, q);
      if (q <= ra2) {
        ++ce;
        cb += (q <= rb2);
        bad |= (q < 1e-12);
      }
    }
  return ce;
}

__global__ void __launch_bounds__(32 * GWPA) k_count(int N, const double *__restrict__ pos,
                                                     const double *__restrict__ frac, const int32_t *__restrict__ soa,
                                                     const int32_t *__restrict__ atom_ptr,
                                                     const StructGeo *__restrict__ geo, double ra2, double rb2,
                                                     int32_t *__restrict__ cnt_e, int32_t *__restrict__ cnt_b,
                                                     int *flag, CellArgs ca) {
  pdl_begin();
  __shared__ int sh[GWPA][2];
  __shared__ int cnt27[28];
  const int i = blockIdx.x, w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (i >= N) return;
  const int s = soa[i];
  const int a0 = atom_ptr[s], a1 = atom_ptr[s + 1];
  const StructGeo &g = geo[s];
  double L[9];
#pragma unroll
  for (int k = 0; k < 9; ++k) L[k] = g.L[k];
  const double fi[3] = {frac[3 * i], frac[3 * i + 1], frac[3 * i + 2]};
  int ce = 0, cbt = 0, bad = 0;
  if (g.nc[0] > 0) {                                  // cell list: candidates of the 27 neighbour cells
    int cc[3];
    cell_prefix(ca, a0, g, ca.atom_cell[i], cnt27, cc);
    const int si[3] = {(int)floor(fi[0]), (int)floor(fi[1]), (int)floor(fi[2])};
    for (int t = threadIdx.x; t < cnt27[27]; t += 32 * GWPA) {
      int j, n1, n2, n3;
      cell_candidate(ca, a0, g, cc[0], cc[1], cc[2], cnt27, t, frac, si, j, n1, n2, n3);
      if (i == j && n1 == 0 && n2 == 0 && n3 == 0) continue;
      double dx, dy, dz, q;
      eval_pair(pos, L, i, j, n1, n2, n3, dx, dy, dz, q);
      if (q <= ra2) {
        ++ce;
        cbt += (q <= rb2);
        bad |= (q < 1e-12);
      }
    }
  } else {
    const int W = (int)floor(2.0 * g.rw[0]) + 4;
    const int nslot = (a1 - a0) * W;
    for (int p = w * 32 + lane; p < nslot; p += 32 * GWPA) {
      int cb, j, n1;
      Range r;
      ce += slot_count(pos, frac, L, g, fi, i, a0, W, p, ra2, rb2, cb, bad, r, j, n1);
      cbt += cb;
    }
  }
  ce = __reduce_add_sync(0xffffffffu, ce);
  cbt = __reduce_add_sync(0xffffffffu, cbt);
  bad = __any_sync(0xffffffffu, bad);
  if (lane == 0) { sh[w][0] = ce; sh[w][1] = cbt; }
  if (bad && lane == 0) atomicOr(flag, 4);
  __syncthreads();
  if (threadIdx.x == 0) {
    int te = 0, tb = 0;
    for (int k = 0; k < GWPA; ++k) { te += sh[k][0]; tb += sh[k][1]; }
    cnt_e[i] = te;
    cnt_b[i] = tb;
  }
}

// single-block exclusive scans of cnt_e, cnt_b and m(m-1); totals (int64) to tot[0..2]
__global__ void k_scan(int N, const int32_t *__restrict__ cnt_e, const int32_t *__restrict__ cnt_b,
                       int32_t *__restrict__ row_ptr, int32_t *__restrict__ bond_ptr,
                       int32_t *__restrict__ ang_ptr, long long *tot) {
  pdl_begin();
  __shared__ long long sh[3][1024];
  int t = threadIdx.x;
  int per = (N + blockDim.x - 1) / blockDim.x;
  int i0 = min(N, t * per), i1 = min(N, i0 + per);
  long long se = 0, sb = 0, sa = 0;
  for (int i = i0; i < i1; ++i) {
    long long m = cnt_b[i];
    se += cnt_e[i]; sb += m; sa += m * (m - 1);
  }
  sh[0][t] = se; sh[1][t] = sb; sh[2][t] = sa;
  __syncthreads();
  for (int off = 1; off < blockDim.x; off <<= 1) {
    long long v0 = 0, v1 = 0, v2 = 0;
    if (t >= off) { v0 = sh[0][t - off]; v1 = sh[1][t - off]; v2 = sh[2][t - off]; }
    __syncthreads();
    sh[0][t] += v0; sh[1][t] += v1; sh[2][t] += v2;
    __syncthreads();
  }
  long long be = sh[0][t] - se, bb = sh[1][t] - sb, ba = sh[2][t] - sa;
  for (int i = i0; i < i1; ++i) {
    long long m = cnt_b[i];
    row_ptr[i] = (int32_t)be; bond_ptr[i] = (int32_t)bb; ang_ptr[i] = (int32_t)ba;
    be += cnt_e[i]; bb += m; ba += m * (m - 1);
  }
  if (t == blockDim.x - 1) {
    tot[0] = sh[0][t]; tot[1] = sh[1][t]; tot[2] = sh[2][t];
    if (sh[0][t] < 2147483647LL && sh[2][t] < 2147483647LL) {
      row_ptr[N] = (int32_t)sh[0][t]; bond_ptr[N] = (int32_t)sh[1][t]; ang_ptr[N] = (int32_t)sh[2][t];
    }
  }
}

__device__ __forceinline__ int warp_excl_scan(int v, int lane, int &total) {
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  total = __shfl_sync(0xffffffffu, x, 31);
  return x - v;
}

// Ordered emission, one 128-thread block per centre atom: rounds of 4 consecutive 32-slot
// chunks (one per warp) — count, block-exclusive scan over the chunks in slot order, then the
// warp-ordered emission of each chunk: the canonical (j, n1, n2, n3) order of the CSR row.
__global__ void __launch_bounds__(32 * GWPA) k_fill(int N, const double *__restrict__ pos,
                                                    const double *__restrict__ frac, const int32_t *__restrict__ soa,
                                                    const int32_t *__restrict__ atom_ptr,
                                                    const StructGeo *__restrict__ geo, double ra2, double rb2,
                                                    const int32_t *__restrict__ row_ptr,
                                                    const int32_t *__restrict__ bond_ptr, int32_t *__restrict__ center,
                                                    int32_t *__restrict__ nbr, char4 *__restrict__ img,
                                                    float4 *__restrict__ vec, double4 *__restrict__ vec64,
                                                    int32_t *__restrict__ bond_id, int32_t *__restrict__ bond_edge,
                                                    CellArgs ca) {
  pdl_begin();
  __shared__ int sh[GWPA][2];
  __shared__ int cnt27[28];
  __shared__ long long keys[CELL_MAXNB];
  __shared__ int nacc, bpre[CELL_MAXNB];
  const int i = blockIdx.x, w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (i >= N) return;
  const int s = soa[i];
  const int a0 = atom_ptr[s], a1 = atom_ptr[s + 1];
  const StructGeo &g = geo[s];
  double L[9];
#pragma unroll
  for (int k = 0; k < 9; ++k) L[k] = g.L[k];
  const double fi[3] = {frac[3 * i], frac[3 * i + 1], frac[3 * i + 2]};
  int be = row_ptr[i], bb = bond_ptr[i];
  if (g.nc[0] > 0 && row_ptr[i + 1] - be <= CELL_MAXNB) {
    // cell list: accepted (j, n) keys collected in any order, sorted (bitonic) into the canonical
    // (j, n1, n2, n3) order of the CSR row, then written with a block scan for the bond numbers
    int cc[3];
    cell_prefix(ca, a0, g, ca.atom_cell[i], cnt27, cc);
    const int si[3] = {(int)floor(fi[0]), (int)floor(fi[1]), (int)floor(fi[2])};
    if (threadIdx.x == 0) nacc = 0;
    __syncthreads();
    for (int t = threadIdx.x; t < cnt27[27]; t += 32 * GWPA) {
      int j, n1, n2, n3;
      cell_candidate(ca, a0, g, cc[0], cc[1], cc[2], cnt27, t, frac, si, j, n1, n2, n3);
      if (i == j && n1 == 0 && n2 == 0 && n3 == 0) continue;
      double dx, dy, dz, q;
      eval_pair(pos, L, i, j, n1, n2, n3, dx, dy, dz, q);
      if (q <= ra2) {
        const int slot = atomicAdd(&nacc, 1);
        if (slot < CELL_MAXNB) keys[slot] = edge_key(j, make_char4((signed char)n1, (signed char)n2, (signed char)n3, 0));
      }
    }
    __syncthreads();
    const int na = min(nacc, CELL_MAXNB);
    int np2 = 1;
    while (np2 < na) np2 <<= 1;
    for (int k = na + threadIdx.x; k < np2; k += 32 * GWPA) keys[k] = 0x7fffffffffffffffLL;
    __syncthreads();
    for (int size = 2; size <= np2; size <<= 1)       // bitonic sort, ascending
      for (int stride = size >> 1; stride > 0; stride >>= 1) {
        for (int k = threadIdx.x; k < np2; k += 32 * GWPA) {
          const int o = k ^ stride;
          if (o > k) {
            const bool up = (k & size) == 0;
            const long long x = keys[k], y = keys[o];
            if ((x > y) == up) { keys[k] = y; keys[o] = x; }
          }
        }
        __syncthreads();
      }
    // bond flags -> exclusive prefix (single thread: <= CELL_MAXNB entries, off the hot path)
    for (int k = threadIdx.x; k < na; k += 32 * GWPA) {
      const long long key = keys[k];
      const int j = (int)(key >> 24);
      const int n1 = (int)((key >> 16) & 255) - 128, n2 = (int)((key >> 8) & 255) - 128, n3 = (int)(key & 255) - 128;
      double dx, dy, dz, q;
      eval_pair(pos, L, i, j, n1, n2, n3, dx, dy, dz, q);
      bpre[k] = q <= rb2;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      int acc = 0;
      for (int k = 0; k < na; ++k) { const int f = bpre[k]; bpre[k] = acc; acc += f; }
    }
    __syncthreads();
    for (int k = threadIdx.x; k < na; k += 32 * GWPA) {
      const long long key = keys[k];
      const int j = (int)(key >> 24);
      const int n1 = (int)((key >> 16) & 255) - 128, n2 = (int)((key >> 8) & 255) - 128, n3 = (int)(key & 255) - 128;
      double dx, dy, dz, q;
      eval_pair(pos, L, i, j, n1, n2, n3, dx, dy, dz, q);
      const int e = be + k;
      center[e] = i;
      nbr[e] = j;
      img[e] = make_char4((signed char)n1, (signed char)n2, (signed char)n3, 0);
      const double rr = sqrt(q);
      vec[e] = make_float4((float)dx, (float)dy, (float)dz, (float)rr);
      vec64[e] = make_double4(dx, dy, dz, rr);
      if (q <= rb2) {
        const int b = bb + bpre[k];
        bond_id[e] = b;
        bond_edge[b] = e;
      } else {
        bond_id[e] = -1;
      }
    }
    return;
  }
  const int W = (int)floor(2.0 * g.rw[0]) + 4;
  const int nslot = (a1 - a0) * W;
  for (int p0 = 0; p0 < nslot; p0 += 32 * GWPA) {
    const int p = p0 + w * 32 + lane;
    int j = 0, n1 = 0, ce = 0, cb = 0, bad = 0;
    Range r;
    if (p < nslot) ce = slot_count(pos, frac, L, g, fi, i, a0, W, p, ra2, rb2, cb, bad, r, j, n1);
    int te, tb;
    const int oe = warp_excl_scan(ce, lane, te);
    const int ob = warp_excl_scan(cb, lane, tb);
    __syncthreads();                                  // previous round's sh reads are done
    if (lane == 0) { sh[w][0] = te; sh[w][1] = tb; }
    __syncthreads();
    int we = be, wb = bb;                             // offsets of this warp's chunk
    for (int k = 0; k < w; ++k) { we += sh[k][0]; wb += sh[k][1]; }
    if (ce > 0) {
      int e = we + oe, b = wb + ob;
      for (int n2 = r.lo[1]; n2 <= r.hi[1]; ++n2)
        for (int n3 = r.lo[2]; n3 <= r.hi[2]; ++n3) {
          if (i == j && n1 == 0 && n2 == 0 && n3 == 0) continue;
          double dx, dy, dz, q;
          eval_pair(pos, L, i, j, n1, n2, n3, dx, dy, dz, q);
          if (q <= ra2) {
            center[e] = i;
            nbr[e] = j;
            img[e] = make_char4((signed char)n1, (signed char)n2, (signed char)n3, 0);
            double rr = sqrt(q);
            vec[e] = make_float4((float)dx, (float)dy, (float)dz, (float)rr);
            vec64[e] = make_double4(dx, dy, dz, rr);
            if (q <= rb2) {
              bond_id[e] = b;
              bond_edge[b] = e;
              ++b;
            } else {
              bond_id[e] = -1;
            }
            ++e;
          }
        }
    }
    for (int k = 0; k < GWPA; ++k) { be += sh[k][0]; bb += sh[k][1]; }
  }
}

__global__ void k_angles(int B, const int32_t *__restrict__ bond_edge, const int32_t *__restrict__ center,
                         const int32_t *__restrict__ bond_ptr, const int32_t *__restrict__ atom_angle_ptr,
                         int32_t *__restrict__ bond_ctr, int32_t *__restrict__ angle_ptr, int32_t *__restrict__ ab1,
                         int32_t *__restrict__ ab2, int32_t *__restrict__ ae1, int32_t *__restrict__ ae2,
                         int32_t *__restrict__ actr, int32_t *__restrict__ swp, int A) {
  pdl_begin();
  int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) {
    if (b == B) angle_ptr[B] = A;
    return;
  }
  int e = bond_edge[b];
  int i = center[e];
  bond_ctr[b] = i;
  int bs = bond_ptr[i], m = bond_ptr[i + 1] - bs, p = b - bs;
  int abase = atom_angle_ptr[i];
  int row = abase + p * (m - 1);
  angle_ptr[b] = row;
  int k = 0;
  for (int q = 0; q < m; ++q) {
    if (q == p) continue;
    int idx = row + k;
    ab1[idx] = b;
    ab2[idx] = bs + q;
    ae1[idx] = e;
    ae2[idx] = bond_edge[bs + q];
    actr[idx] = i;
    swp[idx] = abase + q * (m - 1) + (p < q ? p : p - 1);
    ++k;
  }
}


__global__ void k_rev(int E, const int32_t *__restrict__ center, const int32_t *__restrict__ nbr,
                      const char4 *__restrict__ img, const int32_t *__restrict__ row_ptr,
                      int32_t *__restrict__ rev, int *flag) {
  pdl_begin();
  int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= E) return;
  int i = center[e], j = nbr[e];
  char4 n = img[e];
  char4 mn = make_char4(-n.x, -n.y, -n.z, 0);
  long long key = edge_key(i, mn);
  int lo = row_ptr[j], hi = row_ptr[j + 1] - 1, found = -1;
  while (lo <= hi) {
    int mid = (lo + hi) >> 1;
    long long k = edge_key(nbr[mid], img[mid]);
    if (k == key) { found = mid; break; }
    if (k < key) lo = mid + 1; else hi = mid - 1;
  }
  rev[e] = found;
  if (found < 0) atomicOr(flag, 8);
}

// stable counting sort of atoms by species, one warp (deterministic)
size_t align_up(size_t x) { return (x + 255) & ~size_t(255); }

struct GraphBlocks { void *a = nullptr, *b = nullptr; };

}  // namespace

// ---------------------------------------------------------------------------
// host orchestration
// ---------------------------------------------------------------------------
static uint64_t g_graph_counter = 0;

chg_graph *build_graph_impl(chg_ctx *ctx, int S, const int64_t *atom_ptr, const double *pos,
                            const double *lat, const int32_t *species, double r_atom_model, double r_bond_model,
                            int on_device, int n_species, double skin) {
  if (S < 0 || (S > 0 && (!atom_ptr || !pos || !lat || !species)))
    CHG_THROW(CHG_ERR_ARG, "null input");
  if (!(r_bond_model > 0 && r_bond_model <= r_atom_model) || !std::isfinite(r_atom_model))
    CHG_THROW(CHG_ERR_ARG, "need 0 < r_bond <= r_atom (got %g, %g)", r_atom_model, r_bond_model);
  if (!(skin >= 0.0 && skin < r_atom_model) || !std::isfinite(skin))
    CHG_THROW(CHG_ERR_ARG, "need 0 <= skin < r_atom (got %g)", skin);
  // the lists are built with the list cutoffs r + skin; the model (bases, envelopes) keeps r
  const double r_atom = r_atom_model + skin, r_bond = r_bond_model + skin;
  if (S > 0 && atom_ptr[0] != 0) CHG_THROW(CHG_ERR_ARG, "atom_ptr[0] must be 0");
  for (int s = 0; s < S; ++s)
    if (atom_ptr[s + 1] < atom_ptr[s]) CHG_THROW(CHG_ERR_ARG, "atom_ptr not monotone at %d", s);
  int64_t N = S > 0 ? atom_ptr[S] : 0;
  if (N >= (1LL << 31) / 64) CHG_THROW(CHG_ERR_CAPACITY, "too many atoms (%lld)", (long long)N);
  cudaStream_t st = ctx->stream;

  // per-structure geometry: host inputs are validated here; device inputs by k_geo (no
  // round trip), its errors surface at the size synchronisation below
  const bool dev_geo = on_device && S > 0;
  std::vector<double> L(dev_geo ? 0 : 9 * (size_t)S);
  if (S > 0 && !dev_geo) std::copy(lat, lat + 9 * (size_t)S, L.begin());
  std::vector<StructGeo> geo(S > 0 ? S : 1);
  for (int s = 0; s < S && !dev_geo; ++s) {
    const double *l = &L[9 * s];
    for (int k = 0; k < 9; ++k)
      if (!std::isfinite(l[k])) CHG_THROW(CHG_ERR_GEOMETRY, "structure %d: non-finite lattice", s);
    double det = l[0] * (l[4] * l[8] - l[5] * l[7]) - l[1] * (l[3] * l[8] - l[5] * l[6]) +
                 l[2] * (l[3] * l[7] - l[4] * l[6]);
    double V = std::fabs(det);
    if (!(V > 1e-6)) CHG_THROW(CHG_ERR_GEOMETRY, "structure %d: |det L| = %g", s, V);
    StructGeo &g = geo[s];
    for (int k = 0; k < 9; ++k) g.L[k] = l[k];
    // inverse (row-vector convention: f = r Linv)
    double inv[9] = {l[4] * l[8] - l[5] * l[7], l[2] * l[7] - l[1] * l[8], l[1] * l[5] - l[2] * l[4],
                     l[5] * l[6] - l[3] * l[8], l[0] * l[8] - l[2] * l[6], l[2] * l[3] - l[0] * l[5],
                     l[3] * l[7] - l[4] * l[6], l[1] * l[6] - l[0] * l[7], l[0] * l[4] - l[1] * l[3]};
    for (int k = 0; k < 9; ++k) g.Linv[k] = inv[k] / det;
    for (int k = 0; k < 3; ++k) {
      const double *u = &l[3 * ((k + 1) % 3)], *w = &l[3 * ((k + 2) % 3)];
      double cx = u[1] * w[2] - u[2] * w[1], cy = u[2] * w[0] - u[0] * w[2], cz = u[0] * w[1] - u[1] * w[0];
      double width = V / std::sqrt(cx * cx + cy * cy + cz * cz);
      g.rw[k] = r_atom / width;
      if (g.rw[k] > 100.0) CHG_THROW(CHG_ERR_GEOMETRY, "structure %d: cell too thin for cutoff", s);
    }
    cell_grid(g.rw, atom_ptr[s + 1] - atom_ptr[s], g.nc);
    g.pad = 0;
  }

  chg_graph *G = new chg_graph();
  G->ctx = ctx;
  G->id = ++g_graph_counter;
  G->S = S;
  G->N = N;
  G->r_atom = r_atom_model;
  G->r_bond = r_bond_model;
  G->skin = skin;
  G->atom_ptr_h.assign(atom_ptr, atom_ptr + S + 1);
  if (S == 0) G->atom_ptr_h.assign(1, 0);
  GraphBlocks *bl = new GraphBlocks();
  G->block = bl;

  try {
    // ---- phase 1 allocation: per-atom / per-structure arrays + scratch
    size_t n1 = N + 1;
    size_t sz_atom = align_up(4 * (S + 1)) + align_up(4 * N) * 3 + align_up(4 * n1) * 3 +
                     align_up(4 * (size_t)(n_species + 2)) + align_up(4 * 9 * (size_t)S) +
                     align_up(4 * (size_t)S) + align_up(sizeof(StructGeo) * geo.size()) +
                     align_up(8 * 3 * N) * 2 + align_up(4 * N) * 2 + align_up(64);
    // cell lists only when some structure is large enough to use them (host knows the sizes)
    bool any_cells = false;
    for (int ss = 0; ss < S; ++ss) any_cells = any_cells || atom_ptr[ss + 1] - atom_ptr[ss] >= CELL_MIN;
    if (any_cells) sz_atom += align_up(4 * N) * 4 + align_up(4 * (N + 1));
    void *blk1 = nullptr;
    const auto tm0 = std::chrono::steady_clock::now();
    CUDA_OK(cudaMallocAsync(&blk1, sz_atom, st));
    if (getenv("CHG_GRAPH_TIMING")) {
      const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - tm0).count();
      if (ms > 2.0) fprintf(stderr, "graph build: cudaMallocAsync(blk1 %zu B) %.1f ms\n", sz_atom, ms);
    }
    bl->a = blk1;
    char *c = (char *)blk1;
    auto take = [&](size_t bytes) { void *p = c; c += align_up(bytes); return p; };
    G->atom_ptr = (int32_t *)take(4 * (S + 1));
    G->struct_of_atom = (int32_t *)take(4 * N);
    G->species = (int32_t *)take(4 * N);
    G->row_ptr = (int32_t *)take(4 * n1);
    G->bond_ptr = (int32_t *)take(4 * n1);
    G->atom_angle_ptr = (int32_t *)take(4 * n1);
    G->lattice_f = (float *)take(4 * 9 * (size_t)S);
    G->inv_natoms = (float *)take(4 * (size_t)S);
    StructGeo *d_geo = (StructGeo *)take(sizeof(StructGeo) * geo.size());
    double *d_pos = (double *)take(8 * 3 * N);
    G->pos0 = d_pos;                                  // kept with the graph (skin refresh)
    G->geo_dev = d_geo;
    double *d_frac = (double *)take(8 * 3 * N);
    int32_t *cnt_e = (int32_t *)take(4 * N);
    int32_t *cnt_b = (int32_t *)take(4 * N);
    long long *d_tot = (long long *)take(64);
    CellArgs ca{};
    int32_t *cell_cursor = nullptr;
    if (any_cells) {
      ca.atom_cell = (int32_t *)take(4 * N);
      ca.cell_cnt = (int32_t *)take(4 * N);
      ca.cell_start = (int32_t *)take(4 * (N + 1));
      ca.cell_atoms = (int32_t *)take(4 * N);
      cell_cursor = (int32_t *)take(4 * N);
    }

    // host-side per-atom/per-structure arrays via pinned staging
    size_t hbytes = 4 * (S + 1) + 4 * N + 4 * 9 * (size_t)S + 4 * (size_t)S + sizeof(StructGeo) * geo.size();
    char *h = (char *)ctx->pinned_get(hbytes + 8 * 3 * N + 4 * N);
    char *hp = h;
    int32_t *h_ap = (int32_t *)hp; hp += 4 * (S + 1);
    int32_t *h_soa = (int32_t *)hp; hp += 4 * N;
    float *h_lat = (float *)hp; hp += 4 * 9 * (size_t)S;
    float *h_inv = (float *)hp; hp += 4 * (size_t)S;
    StructGeo *h_geo = (StructGeo *)hp; hp += sizeof(StructGeo) * geo.size();
    for (int s = 0; s <= S; ++s) h_ap[s] = (int32_t)G->atom_ptr_h[s];
    for (int s = 0; s < S; ++s) {
      for (int64_t a = atom_ptr[s]; a < atom_ptr[s + 1]; ++a) h_soa[a] = s;
      if (!dev_geo)
        for (int k = 0; k < 9; ++k) h_lat[9 * s + k] = (float)L[9 * s + k];
      int64_t ns = atom_ptr[s + 1] - atom_ptr[s];
      h_inv[s] = ns > 0 ? 1.0f / (float)ns : 0.0f;
    }
    std::copy(geo.begin(), geo.end(), h_geo);
    CUDA_OK(cudaMemcpyAsync(G->atom_ptr, h_ap, 4 * (S + 1), cudaMemcpyHostToDevice, st));
    if (N) CUDA_OK(cudaMemcpyAsync(G->struct_of_atom, h_soa, 4 * N, cudaMemcpyHostToDevice, st));
    if (S) {
      if (!dev_geo) CUDA_OK(cudaMemcpyAsync(G->lattice_f, h_lat, 4 * 9 * (size_t)S, cudaMemcpyHostToDevice, st));
      CUDA_OK(cudaMemcpyAsync(G->inv_natoms, h_inv, 4 * (size_t)S, cudaMemcpyHostToDevice, st));
    }
    if (!dev_geo) CUDA_OK(cudaMemcpyAsync(d_geo, h_geo, sizeof(StructGeo) * geo.size(), cudaMemcpyHostToDevice, st));
    if (N) {
      if (on_device) {
        CUDA_OK(cudaMemcpyAsync(d_pos, pos, 8 * 3 * N, cudaMemcpyDeviceToDevice, st));
        CUDA_OK(cudaMemcpyAsync(G->species, species, 4 * N, cudaMemcpyDeviceToDevice, st));
      } else {
        double *hpos = (double *)hp;
        int32_t *hsp = (int32_t *)(hp + 8 * 3 * N);
        std::copy(pos, pos + 3 * N, hpos);
        std::copy(species, species + N, hsp);
        CUDA_OK(cudaMemcpyAsync(d_pos, hpos, 8 * 3 * N, cudaMemcpyHostToDevice, st));
        CUDA_OK(cudaMemcpyAsync(G->species, hsp, 4 * N, cudaMemcpyHostToDevice, st));
      }
    }
    int *flag = ctx->d_flag;
    std::optional<ProfScope> ps1;        // device work only: closed before the host synchronisation
    ps1.emplace(ctx, "graph", 0.0, 0.0);
    CUDA_OK(cudaMemsetAsync(flag, 0, sizeof(int), st));
    CUDA_OK(cudaMemsetAsync(flag + 1, 0x7f, sizeof(int), st));       // smallest bad structure (k_geo)
    CUDA_OK(cudaMemsetAsync(d_tot, 0, 64, st));
    double ra2 = r_atom * r_atom, rb2 = r_bond * r_bond;
    if (dev_geo) {
      launch_k(ctx, k_geo, ceil_div(S, 128), 128, 0, st, S, lat, r_atom, G->atom_ptr, d_geo, G->lattice_f, flag);
      check_launch(ctx);
    }
    if (N) {
      launch_k(ctx, k_frac, ceil_div(N, 256), 256, 0, st, (int)N, d_pos, G->struct_of_atom, d_geo, G->species,
                                                n_species, d_frac, flag);
      check_launch(ctx);
      if (any_cells) {
        CUDA_OK(cudaMemsetAsync(ca.cell_cnt, 0, 4 * N, st));
        CUDA_OK(cudaMemsetAsync(cell_cursor, 0, 4 * N, st));
        launch_k(ctx, k_cell_assign, ceil_div(N, 256), 256, 0, st, (int)N, d_frac, G->struct_of_atom, G->atom_ptr, d_geo, ca);
        check_launch(ctx);
        launch_k(ctx, k_cell_scan, S, 256, 0, st, S, G->atom_ptr, d_geo, ca);
        check_launch(ctx);
        launch_k(ctx, k_cell_place, ceil_div(N, 256), 256, 0, st, (int)N, G->struct_of_atom, G->atom_ptr, ca, cell_cursor);
        check_launch(ctx);
      }
      launch_k(ctx, k_count, (unsigned)N, 32 * GWPA, 0, st, (int)N, d_pos, d_frac, G->struct_of_atom, G->atom_ptr,
                                                      d_geo, ra2, rb2, cnt_e, cnt_b, flag, ca);
      check_launch(ctx);
      launch_k(ctx, k_scan, 1, 1024, 0, st, (int)N, cnt_e, cnt_b, G->row_ptr, G->bond_ptr, G->atom_angle_ptr, d_tot);
      check_launch(ctx);
    } else {
      CUDA_OK(cudaMemsetAsync(G->row_ptr, 0, 4, st));
      CUDA_OK(cudaMemsetAsync(G->bond_ptr, 0, 4, st));
      CUDA_OK(cudaMemsetAsync(G->atom_angle_ptr, 0, 4, st));
    }
    ps1.reset();
    // totals + flags to host (the one synchronisation of the build: sizes)
    long long *h_tot = (long long *)ctx->pinned_get(64);
    CUDA_OK(cudaMemcpyAsync(h_tot, d_tot, 32, cudaMemcpyDeviceToHost, st));
    CUDA_OK(cudaMemcpyAsync(((char *)h_tot) + 32, flag, 2 * sizeof(int), cudaMemcpyDeviceToHost, st));
    static const bool gtime = getenv("CHG_GRAPH_TIMING") != nullptr;   // debug: slow size readbacks
    const auto tq0 = std::chrono::steady_clock::now();
    CUDA_OK(cudaStreamSynchronize(st));
    if (gtime) {
      const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - tq0).count();
      if (ms > 5.0) fprintf(stderr, "graph build: size readback waited %.1f ms (N %lld)\n", ms, (long long)N);
    }
    int hflag = *(int *)(((char *)h_tot) + 32), hbad = *(int *)(((char *)h_tot) + 36);
    if (hflag & 16) CHG_THROW(CHG_ERR_GEOMETRY, "structure %d: non-finite lattice", hbad);
    if (hflag & 32) CHG_THROW(CHG_ERR_GEOMETRY, "structure %d: |det L| <= 1e-6", hbad);
    if (hflag & 64) CHG_THROW(CHG_ERR_GEOMETRY, "structure %d: cell too thin for cutoff", hbad);
    if (hflag & 1) CHG_THROW(CHG_ERR_GEOMETRY, "non-finite positions");
    if (hflag & 2) CHG_THROW(CHG_ERR_SPECIES, "species outside 1..%d", n_species);
    if (hflag & 4) CHG_THROW(CHG_ERR_GEOMETRY, "coincident atoms (accepted pair with d^2 < 1e-12)");
    long long E = h_tot[0], B = h_tot[1], A = h_tot[2];
    if (E >= 2147483647LL || A >= 2147483647LL)
      CHG_THROW(CHG_ERR_CAPACITY, "edge/angle count exceeds int32 (E=%lld A=%lld)", E, A);
    G->E = E; G->B = B; G->A = A;

    // ---- phase 2 allocation: edge / bond / angle arrays
    size_t sz2 = align_up(4 * E) * 4 + align_up(4 * E) /*img*/ + align_up(16 * E) + align_up(32 * E) + align_up(4 * B) * 2 +
                 align_up(4 * (B + 1)) + align_up(4 * A) * 6 + align_up(16) + 256;
    void *blk2 = nullptr;
    const auto tm1 = std::chrono::steady_clock::now();
    CUDA_OK(cudaMallocAsync(&blk2, sz2, st));
    if (getenv("CHG_GRAPH_TIMING")) {
      const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - tm1).count();
      if (ms > 2.0) fprintf(stderr, "graph build: cudaMallocAsync(blk2 %zu B) %.1f ms\n", sz2, ms);
    }
    bl->b = blk2;
    c = (char *)blk2;
    G->center = (int32_t *)take(4 * E);
    G->nbr = (int32_t *)take(4 * E);
    G->bond_id = (int32_t *)take(4 * E);
    G->rev = (int32_t *)take(4 * E);
    G->img = (char4 *)take(4 * E);
    G->vec = (float4 *)take(16 * E);
    G->vec64 = (double4 *)take(32 * E);
    G->bond_edge = (int32_t *)take(4 * B);
    G->bond_ctr = (int32_t *)take(4 * B);
    G->angle_ptr = (int32_t *)take(4 * (B + 1));
    G->angle_b1 = (int32_t *)take(4 * A);
    G->angle_b2 = (int32_t *)take(4 * A);
    G->angle_e1 = (int32_t *)take(4 * A);
    G->angle_e2 = (int32_t *)take(4 * A);
    G->angle_ctr = (int32_t *)take(4 * A);
    G->swap = (int32_t *)take(4 * A);
    G->d_flag = (int *)take(16);
    CUDA_OK(cudaMemsetAsync(G->d_flag, 0, 16, st));

    ProfScope ps2(ctx, "graph", 0.0, 0.0);
    if (N) {
      launch_k(ctx, k_fill, (unsigned)N, 32 * GWPA, 0, st, (int)N, d_pos, d_frac, G->struct_of_atom, G->atom_ptr,
                                                     d_geo, ra2, rb2, G->row_ptr, G->bond_ptr, G->center,
                                                     G->nbr, G->img, G->vec, G->vec64, G->bond_id, G->bond_edge, ca);
      check_launch(ctx);
      launch_k(ctx, k_angles, ceil_div(B + 1, 256), 256, 0, st, (int)B, G->bond_edge, G->center, G->bond_ptr,
                                                      G->atom_angle_ptr, G->bond_ctr, G->angle_ptr, G->angle_b1,
                                                      G->angle_b2, G->angle_e1, G->angle_e2, G->angle_ctr,
                                                      G->swap, (int)A);
      check_launch(ctx);
      if (E) {
        launch_k(ctx, k_rev, ceil_div(E, 256), 256, 0, st, (int)E, G->center, G->nbr, G->img, G->row_ptr, G->rev, G->d_flag);
        check_launch(ctx);
      }

    } else {
      CUDA_OK(cudaMemsetAsync(G->angle_ptr, 0, 4, st));
    }
  } catch (...) {
    if (bl->a) cudaFreeAsync(bl->a, st);
    if (bl->b) cudaFreeAsync(bl->b, st);
    delete bl;
    delete G;
    throw;
  }
  CUDA_OK(cudaEventCreateWithFlags(&G->ready, cudaEventDisableTiming));
  CUDA_OK(cudaEventRecord(G->ready, st));
  return G;
}

// ---------------------------------------------------------------------------
// fixed-topology refresh (skin graphs, captured MD steps): every edge's geometry from the new
// positions by the same canonical fp64 evaluation as the build (bit-identical to a fresh
// build's value for that pair); the lists, bond flags and angles stay those of the build
// ---------------------------------------------------------------------------
__global__ void k_refresh(int E, const double *__restrict__ pos, const StructGeo *__restrict__ geo,
                          const int32_t *__restrict__ soa, const int32_t *__restrict__ center,
                          const int32_t *__restrict__ nbr, const char4 *__restrict__ img, float4 *__restrict__ vec,
                          double4 *__restrict__ vec64) {
  pdl_begin();
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= E) return;
  const int i = center[e], j = nbr[e];
  const char4 n = img[e];
  double dx, dy, dz, q;
  eval_pair(pos, geo[soa[i]].L, i, j, n.x, n.y, n.z, dx, dy, dz, q);
  const double rr = sqrt(q);
  vec[e] = make_float4((float)dx, (float)dy, (float)dz, (float)rr);
  vec64[e] = make_double4(dx, dy, dz, rr);
}

// flag <- 1 when some atom moved more than skin / 2 since the build (the Verlet-list bound:
// then a pair may have crossed the model cutoff without being in the lists)
__global__ void k_moved(int N, const double *__restrict__ pos, const double *__restrict__ pos0, double lim2,
                        int32_t *__restrict__ flag) {
  pdl_begin();
  const int a = blockIdx.x * blockDim.x + threadIdx.x;
  if (a >= N) return;
  const double dx = pos[3 * a] - pos0[3 * a], dy = pos[3 * a + 1] - pos0[3 * a + 1], dz = pos[3 * a + 2] - pos0[3 * a + 2];
  if (dx * dx + dy * dy + dz * dz > lim2) *flag = 1;
}

void graph_refresh(chg_ctx *ctx, chg_graph *G, const double *pos, int32_t *flag) {
  if (!G->geo_dev || !G->pos0) CHG_THROW(CHG_ERR_STATE, "graph has no build geometry");
  const int64_t E = G->E, N = G->N;
  ProfScope ps(ctx, "graph_refresh", 0.0, 64.0 * E + 48.0 * N);
  if (E) {
    launch_k(ctx, k_refresh, ceil_div(E, 256), 256, 0, ctx->stream, (int)E, pos, (const StructGeo *)G->geo_dev,
             G->struct_of_atom, G->center, G->nbr, G->img, G->vec, G->vec64);
    check_launch(ctx);
  }
  if (flag && N) {
    const double h = 0.5 * G->skin;
    launch_k(ctx, k_moved, ceil_div(N, 256), 256, 0, ctx->stream, (int)N, pos, G->pos0, h * h, flag);
    check_launch(ctx);
  }
}

// Per-structure counts (chg_graph_counts) read on demand: the build itself synchronises
// only once (for the array sizes).  Also surfaces the reverse-edge invariant flag.
void graph_fill_counts(chg_graph *G) {
  const int S = G->S;
  const int64_t N = G->N;
  chg_ctx *ctx = G->ctx;
  cudaStream_t st = ctx->stream;
  G->counts_h.assign(4 * (size_t)S, 0);
  if (!S) return;
  int32_t *hrp = (int32_t *)ctx->pinned_get(4 * (N + 1) * 3 + 64);
  CUDA_OK(cudaMemcpyAsync(hrp, G->row_ptr, 4 * (N + 1), cudaMemcpyDeviceToHost, st));
  CUDA_OK(cudaMemcpyAsync(hrp + (N + 1), G->bond_ptr, 4 * (N + 1), cudaMemcpyDeviceToHost, st));
  CUDA_OK(cudaMemcpyAsync(hrp + 2 * (N + 1), G->atom_angle_ptr, 4 * (N + 1), cudaMemcpyDeviceToHost, st));
  hrp[3 * (N + 1)] = 0;
  if (G->d_flag) CUDA_OK(cudaMemcpyAsync(hrp + 3 * (N + 1), G->d_flag, 4, cudaMemcpyDeviceToHost, st));
  CUDA_OK(cudaStreamSynchronize(st));
  if (hrp[3 * (N + 1)] & 8) CHG_THROW(CHG_ERR_GEOMETRY, "internal: reverse edge not found");
  for (int s = 0; s < S; ++s) {
    int64_t a0 = G->atom_ptr_h[s], a1 = G->atom_ptr_h[s + 1];
    G->counts_h[4 * s + 0] = a1 - a0;
    G->counts_h[4 * s + 1] = hrp[a1] - hrp[a0];
    G->counts_h[4 * s + 2] = hrp[N + 1 + a1] - hrp[N + 1 + a0];
    G->counts_h[4 * s + 3] = hrp[2 * (N + 1) + a1] - hrp[2 * (N + 1) + a0];
  }
  G->counts_ready = true;
}

void destroy_graph_impl(chg_graph *G) {
  if (!G) return;
  if (G->user && G->user != G->ctx) {          // used on another context's stream: free after its work
    cudaEvent_t done;
    if (cudaEventCreateWithFlags(&done, cudaEventDisableTiming) == cudaSuccess) {
      cudaEventRecord(done, G->user->stream);
      cudaStreamWaitEvent(G->ctx->stream, done, 0);
      cudaEventDestroy(done);
    }
  }
  if (G->ready) cudaEventDestroy(G->ready);
  if (G->block) {
    GraphBlocks *bl = (GraphBlocks *)G->block;
    if (bl->a) cudaFreeAsync(bl->a, G->ctx->stream);
    if (bl->b) cudaFreeAsync(bl->b, G->ctx->stream);
    delete bl;
  }
  delete G;
}
