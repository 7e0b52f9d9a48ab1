// pf_device.cuh — device-side building blocks of the B200 phase-field hot path (sm_100a, FP64).
//
//  * DMesh / Consts: the structured row-compact mesh (include/pf_b200.h: pf_mesh) and the
//    per-handle constants, passed BY VALUE as kernel parameters (constant bank) so several
//    handles with different meshes can coexist in one process.
//  * Q4 element math on uniform square cells using the tensor-product structure of the 2x2
//    Gauss rule: d/dx at a Gauss point depends only on its eta, d/dy only
//    on its xi, so each derivative takes two distinct values per element.
//  * Deterministic reductions (fixed-order warp butterflies, block trees, per-CTA partials).
//
// Reference formulas restated here (file:line under /root/reference/pkg/src/phasefrac):
//   strain / Voigt invariants      assembly.py:152-158, material.py:107-116
//   degraded stress                material.py:162-176 (macaulay :119-126, g(d) :129-138)
//   tangent                        material.py:185-201
//   evolution residual / tangent   assembly.py:217-246, material.py:85-96
//   gate / extra stiffness         schemes.py:96-142
//   active-energy update           schemes.py:145-176
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace pfb {

constexpr int TX = 32;   // owned node columns per tile (one warp row -> 512 B coalesced rows)
constexpr int TY = 8;    // owned node rows per tile
constexpr int NT = 256;  // threads per CTA for tile kernels
constexpr int HX = TX + 2, HY = TY + 2;  // node halo region
constexpr int EX = TX + 1, EY = TY + 1;  // cell region (every cell touching an owned node)

struct DMesh {
  int nx, ny;
  const int* nlo;   // [ny+1]
  const int* nhi;
  const int* nst;
  const int* elo;   // [ny]
  const int* ehi;
  const int* est;
  int notch_row, notch_lo, notch_hi, dup_start;  // notch_row = -1: none
  int n_nodes, n_elems;
  int n_tiles;
  const int2* tiles;  // active tile coordinates (tile column, tile row)
  const int4* nrow;   // [ny+1] packed (lo, hi, start, 0) of node rows
  const int4* erow;   // [ny]   packed (lo, hi, start, 0) of cell rows
  // ownership (row-strip decomposition): owned nodes are [own_lo, own_hi) plus [dup_lo, n);
  // owned cells [cell_lo, cell_hi).  Single GPU: everything owned.
  int own_lo, own_hi, dup_lo, cell_lo, cell_hi;
};

__device__ __forceinline__ bool node_owned(const DMesh& m, int id) {
  return (id >= m.own_lo && id < m.own_hi) || id >= m.dup_lo;
}
__device__ __forceinline__ bool cell_owned(const DMesh& m, int eid) {
  return eid >= m.cell_lo && eid < m.cell_hi;
}

struct Consts {
  double Px, Mx, Py, My;      // (1 + c)/(2 hx), (1 - c)/(2 hx), same with hy; c = 1/sqrt(3)
  double Pxw, Mxw, Pyw, Myw;  // times wdet
  double P2xw, M2xw, P2yw, M2yw;  // squares times wdet
  double w;           // wdet = det J * weight = hx*hy/4
  double N[4][4];     // N[g][a] shape values (assembly.py:33-43, _GP order :28)
  double Nw[4][4];    // N[g][a] * wdet
  double lap[4][4];   // grad_w * sum_g gradN_a . gradN_b * wdet
  double mu, k, two_mu, mu43;  // mu43 = 2 mu (1 - 1/3): tangent normal diagonal
  double third;                // 1/3 (tangent apply only; residuals divide like the reference)
  double eta, gamma, src_base, grad_w, psi_crit, d_cap;
  int at2;
};

// ----------------------------------------------------------------------------------------
// cache-policy loads: data written inside a persistent kernel by other CTAs must bypass L1
__device__ __forceinline__ double ldcg(const double* p) { return __ldcg(p); }
__device__ __forceinline__ double2 ldcg(const double2* p) { return __ldcg(p); }
__device__ __forceinline__ double ldro(const double* p) { return __ldg(p); }
__device__ __forceinline__ double2 ldro(const double2* p) { return __ldg(p); }

// ----------------------------------------------------------------------------------------
// deterministic reductions
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;  // butterfly: every lane holds bit-identical totals
}

// Block-wide sum of NV values; result valid in thread 0. `red` holds NT/32*NV doubles.
// Lane's ordered partial sum of part[stride * i + k] over i = lane, lane + 32, ... < n: the
// loads of LANE_SUM_BATCH rows are issued before their adds, so a grid-wide reduction costs one
// L2 round trip per batch instead of one per row (the additions, and so the bits, are those of
// the plain loop).
constexpr int LANE_SUM_BATCH = 4;
template <int NV>
__device__ __forceinline__ void lane_ordered_sum(const double* part, int stride, int n,
                                                 double (&s)[NV]) {
  constexpr int B = NV <= 3 ? LANE_SUM_BATCH : 1;  // (wide partial rows: registers)
  for (int base = (int)(threadIdx.x & 31); base < n; base += 32 * B) {
    double v[B][NV];
#pragma unroll
    for (int q = 0; q < B; ++q) {
      const int i = base + 32 * q;
#pragma unroll
      for (int k = 0; k < NV; ++k) v[q][k] = i < n ? __ldcg(part + (size_t)stride * i + k) : 0.0;
    }
#pragma unroll
    for (int q = 0; q < B; ++q)
      if (base + 32 * q < n) {
#pragma unroll
        for (int k = 0; k < NV; ++k) s[k] += v[q][k];
      }
  }
}

template <int NV>
__device__ __forceinline__ void block_sum(double (&v)[NV], double* red) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < NV; ++k) v[k] = warp_sum(v[k]);
  if (lane == 0) {
#pragma unroll
    for (int k = 0; k < NV; ++k) red[wid * NV + k] = v[k];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      double s = 0.0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += red[w * NV + k];
      v[k] = s;
    }
  }
  __syncthreads();
}

// ----------------------------------------------------------------------------------------
// per-tile row tables (node rows ty0-1 .. ty0+TY, cell rows ty0-1 .. ty0+TY-1)
struct TileRows {
  int nlo[HY], nhi[HY], nst[HY];
  int elo[EY], ehi[EY], est[EY];
};

__device__ __forceinline__ void load_tile_rows(const DMesh& m, int ty0, TileRows& R) {
  const int t = threadIdx.x;
  if (t < HY) {
    const int j = ty0 - 1 + t;
    if (j >= 0 && j <= m.ny) {
      R.nlo[t] = __ldg(m.nlo + j); R.nhi[t] = __ldg(m.nhi + j); R.nst[t] = __ldg(m.nst + j);
    } else {
      R.nlo[t] = 0; R.nhi[t] = 0; R.nst[t] = 0;
    }
  } else if (t >= 32 && t < 32 + EY) {
    const int e = t - 32, j = ty0 - 1 + e;
    if (j >= 0 && j < m.ny) {
      R.elo[e] = __ldg(m.elo + j); R.ehi[e] = __ldg(m.ehi + j); R.est[e] = __ldg(m.est + j);
    } else {
      R.elo[e] = 0; R.ehi[e] = 0; R.est[e] = 0;
    }
  }
}

__device__ __forceinline__ int tile_node(const TileRows& R, int hy, int i) {
  return (i >= R.nlo[hy] && i < R.nhi[hy]) ? R.nst[hy] + (i - R.nlo[hy]) : -1;
}
__device__ __forceinline__ int tile_cell(const TileRows& R, int ey, int ci) {
  return (ci >= R.elo[ey] && ci < R.ehi[ey]) ? R.est[ey] + (ci - R.elo[ey]) : -1;
}
__device__ __forceinline__ bool is_dup_col(const DMesh& m, int i) {
  return i >= m.notch_lo && i < m.notch_hi;
}

// global (non-tile) lookups
__device__ __forceinline__ int node_at(const DMesh& m, int i, int j) {
  if (j < 0 || j > m.ny) return -1;
  const int lo = __ldg(m.nlo + j), hi = __ldg(m.nhi + j);
  return (i >= lo && i < hi) ? __ldg(m.nst + j) + (i - lo) : -1;
}
// the four node ids of cell (ci, cj) (caller checked that the cell exists)
__device__ __forceinline__ void cell_nodes(const DMesh& m, int ci, int cj, int (&n)[4]) {
  n[0] = node_at(m, ci, cj);
  n[1] = node_at(m, ci + 1, cj);
  n[2] = node_at(m, ci + 1, cj + 1);
  n[3] = node_at(m, ci, cj + 1);
  if (cj == m.notch_row) {
    if (is_dup_col(m, ci)) n[0] = m.dup_start + (ci - m.notch_lo);
    if (is_dup_col(m, ci + 1)) n[1] = m.dup_start + (ci + 1 - m.notch_lo);
  }
}
__device__ __forceinline__ int cell_at(const DMesh& m, int ci, int cj) {
  if (cj < 0 || cj >= m.ny) return -1;
  const int lo = __ldg(m.elo + cj), hi = __ldg(m.ehi + cj);
  return (ci >= lo && ci < hi) ? __ldg(m.est + cj) + (ci - lo) : -1;
}

// ----------------------------------------------------------------------------------------
// Q4 kinematics on a uniform rectangular cell (hx x hy).
// Corners 0..3 CCW from (-,-); Gauss points g0..g3 = (-,-),(+,-),(+,+),(-,+)/sqrt(3).
struct Strain4 {
  double exx[4], eyy[4], gxy[4];
};

__device__ __forceinline__ void strain_q4(const Consts& C, double2 u0, double2 u1, double2 u2,
                                          double2 u3, Strain4& s) {
  const double bx = u1.x - u0.x, tx = u2.x - u3.x;  // ux jump along x: bottom / top edge
  const double by = u1.y - u0.y, ty = u2.y - u3.y;  // uy jump along x
  const double lx = u3.x - u0.x, rx = u2.x - u1.x;  // ux jump along y: left / right edge
  const double ly = u3.y - u0.y, ry = u2.y - u1.y;  // uy jump along y
  const double uxx_lo = C.Px * bx + C.Mx * tx, uxx_hi = C.Mx * bx + C.Px * tx;  // eta = -c/+c
  const double uyx_lo = C.Px * by + C.Mx * ty, uyx_hi = C.Mx * by + C.Px * ty;
  const double uxy_l = C.Py * lx + C.My * rx, uxy_r = C.My * lx + C.Py * rx;    // xi = -c/+c
  const double uyy_l = C.Py * ly + C.My * ry, uyy_r = C.My * ly + C.Py * ry;
  s.exx[0] = uxx_lo; s.exx[1] = uxx_lo; s.exx[2] = uxx_hi; s.exx[3] = uxx_hi;
  s.eyy[0] = uyy_l;  s.eyy[1] = uyy_r;  s.eyy[2] = uyy_r;  s.eyy[3] = uyy_l;
  s.gxy[0] = uxy_l + uyx_lo; s.gxy[1] = uxy_r + uyx_lo;
  s.gxy[2] = uxy_r + uyx_hi; s.gxy[3] = uxy_l + uyx_hi;
}

// f_a = sum_g B_a(g)^T sigma_g wdet for in-plane stress (xx, yy, xy) at the 4 Gauss points.
__device__ __forceinline__ void backproject_q4(const Consts& C, const double (&sxx)[4],
                                               const double (&syy)[4], const double (&sxy)[4],
                                               double2 (&f)[4]) {
  auto SA = [&](const double (&s)[4]) { return C.Pxw * (s[0] + s[1]) + C.Mxw * (s[2] + s[3]); };
  auto SB = [&](const double (&s)[4]) { return C.Mxw * (s[0] + s[1]) + C.Pxw * (s[2] + s[3]); };
  auto SC = [&](const double (&s)[4]) { return C.Pyw * (s[0] + s[3]) + C.Myw * (s[1] + s[2]); };
  auto SD = [&](const double (&s)[4]) { return C.Myw * (s[0] + s[3]) + C.Pyw * (s[1] + s[2]); };
  const double axx = SA(sxx), bxx = SB(sxx);
  const double cyy = SC(syy), dyy = SD(syy);
  const double axy = SA(sxy), bxy = SB(sxy), cxy = SC(sxy), dxy = SD(sxy);
  f[0] = make_double2(-axx - cxy, -cyy - axy);
  f[1] = make_double2(axx - dxy, -dyy + axy);
  f[2] = make_double2(bxx + dxy, dyy + bxy);
  f[3] = make_double2(-bxx + cxy, cyy - bxy);
}

// diagonal of sum_g B^T C_g B wdet with C_g = [[lam, ., 0],[., lam, 0],[0, 0, sh]]
__device__ __forceinline__ void diag_q4(const Consts& C, const double (&lam)[4],
                                        const double (&sh)[4], double2 (&dg)[4]) {
  auto QA = [&](const double (&v)[4]) { return C.P2xw * (v[0] + v[1]) + C.M2xw * (v[2] + v[3]); };
  auto QB = [&](const double (&v)[4]) { return C.M2xw * (v[0] + v[1]) + C.P2xw * (v[2] + v[3]); };
  auto QC = [&](const double (&v)[4]) { return C.P2yw * (v[0] + v[3]) + C.M2yw * (v[1] + v[2]); };
  auto QD = [&](const double (&v)[4]) { return C.M2yw * (v[0] + v[3]) + C.P2yw * (v[1] + v[2]); };
  const double la = QA(lam), lb = QB(lam), lc = QC(lam), ld = QD(lam);
  const double sa = QA(sh), sb = QB(sh), sc = QC(sh), sd = QD(sh);
  dg[0] = make_double2(la + sc, lc + sa);
  dg[1] = make_double2(la + sd, ld + sa);
  dg[2] = make_double2(lb + sd, ld + sb);
  dg[3] = make_double2(lb + sc, lc + sb);
}

__device__ __forceinline__ void interp_q4(const Consts& C, double v0, double v1, double v2,
                                          double v3, double (&out)[4]) {
#pragma unroll
  for (int g = 0; g < 4; ++g)
    out[g] = C.N[g][0] * v0 + C.N[g][1] * v1 + C.N[g][2] * v2 + C.N[g][3] * v3;
}

__device__ __forceinline__ double degradation(const Consts& C, double d) {
  const double om = 1.0 - d;
  return om * om + C.eta;  // material.py:136
}

// Degraded stress (in-plane rows) and the tangent branch flag at one Gauss point.
__device__ __forceinline__ void stress_gp(const Consts& C, double exx, double eyy, double gxy,
                                          double g, double& sxx, double& syy, double& sxy,
                                          bool& plus) {
  const double tr = exx + eyy;           // eps_zz = 0 (plane strain)
  const double at = fabs(tr);
  const double trp = 0.5 * (tr + at), trm = 0.5 * (tr - at);  // macaulay, material.py:119-126
  const double t3 = tr / 3.0;
  sxx = (C.two_mu * (exx - t3) + C.k * trp) * g + C.k * trm;
  syy = (C.two_mu * (eyy - t3) + C.k * trp) * g + C.k * trm;
  sxy = (C.mu * gxy) * g;
  plus = tr >= 0.0;  // material.py:193: tensile branch at tr == 0
}

// Tangent-vector product at one Gauss point: sigma = C(u, d) : eps(p)
__device__ __forceinline__ void tangent_gp(const Consts& C, double exx, double eyy, double gxy,
                                           double g, bool plus, double& sxx, double& syy,
                                           double& sxy) {
  const double tr = exx + eyy, t3 = tr / 3.0;
  const double kv = plus ? g * C.k : C.k;
  const double g2mu = g * C.two_mu;
  sxx = g2mu * (exx - t3) + kv * tr;
  syy = g2mu * (eyy - t3) + kv * tr;
  sxy = g * C.mu * gxy;
}

// GP invariants from strain (material.py:107-116, assembly.py:265-269)
__device__ __forceinline__ void invariants_gp(const Consts& C, double exx, double eyy,
                                              double gxy, double& tr, double& trp,
                                              double& dev2, double& psi) {
  tr = exx + eyy;
  const double t3 = tr / 3.0;
  const double dxx = exx - t3, dyy = eyy - t3, dzz = 0.0 - t3;
  dev2 = dxx * dxx + dyy * dyy + dzz * dzz + 0.5 * gxy * gxy;
  trp = 0.5 * (tr + fabs(tr));
  psi = C.mu * dev2 + 0.5 * C.k * trp * trp;
}

// Fast-scheme gate (schemes.py:96-109)
__device__ __forceinline__ bool gate_gp(const Consts& C, double psi, double psimax, double dg) {
  return (psi > C.psi_crit) && (psi > psimax) && (dg < C.d_cap);
}

// extra stiffness multiplier -4 (1-d)^2/g * X (schemes.py:131-141); scheme 1=S1,2=S2,3=S3
__device__ __forceinline__ double extra_gp(const Consts& C, int scheme, double dg, double trp,
                                           double dev2) {
  const double g = degradation(C, dg);
  const double om = 1.0 - dg;
  const double base = -4.0 * (om * om) / g;
  const double vol = C.k * (trp * trp);
  const double dev = C.two_mu * dev2;
  const double x = scheme == 1 ? vol : (scheme == 2 ? dev : vol + dev);
  return base * x;
}

}  // namespace pfb
