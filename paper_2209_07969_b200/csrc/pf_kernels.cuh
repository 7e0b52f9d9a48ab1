// pf_kernels.cuh — sm_100a FP64 kernels of the staggered phase-field hot path.
//
// Layout in HBM (reference layouts, no permutation at the boundary):
//   u, R_u, x_u, r_u, q_u, p_u, Dinv_u : double2 per node (ux, uy)      assembly.py:132-134
//   d, d_prev, R_d, x_d, ...           : double per node
//   GP arrays (tr+, dev.dev, psi+, psi_max, b) : double[4] per element  assembly.py:46-72
//   flags_u                            : uint8 per element, bit g = [tr eps(u) >= 0] at GP g
//   umask (uint8 per u-DOF) / pmask (uint8 per node): 1 = free DOF
//
// Operators are matrix-free.  Every node-valued output is produced by the tile that OWNS the
// node: a CTA loads its TXxTY node tile plus a one-node halo into shared memory, evaluates every
// cell touching an owned node once, stores per-corner cell contributions in shared memory and
// sums the (up to) four contributions of each owned node in a fixed order -> bit-reproducible
// results without atomics (SURVEY.md §7 hard part 6).
#pragma once
#include <cooperative_groups.h>

#include "pf_device.cuh"

namespace pfb {
namespace cg = cooperative_groups;
static_assert(NT == TX * TY, "tile kernels map one owned node per thread");

// ========================================================================================
// shared-memory images
struct SmemVec2Tile {          // momentum (double2 nodal field + nodal d)
  TileRows R;
  double2 p[HY][HX];
  double2 pdup[HX];
  double d[HY][HX];
  double ddup[HX];
  double2 f[4][EY][EX];        // per-corner cell contributions (SoA over corners)
  double red[NT / 32 * 4];
};

struct SmemScalTile {          // phase field (double nodal fields)
  TileRows R;
  double p[HY][HX];
  double pdup[HX];
  double a[HY][HX];            // second nodal field (d_prev for the residual)
  double adup[HX];
  double f[4][EY][EX];
  double red[NT / 32 * 4];
};

// node slots of the tile: 0..HX*HY-1 = halo grid, HX*HY..HX*HY+HX-1 = duplicate (notch) row
struct Slot {
  int id;        // node id or -1
  bool owned;
  int hx, hy;    // hy = -1 for the dup row
};

__device__ __forceinline__ bool tile_has_dup(const DMesh& m, int ty0) {
  // cells of row notch_row lie in the cell region iff notch_row in [ty0-1, ty0+TY-1]
  return m.notch_row >= 0 && m.notch_row >= ty0 - 1 && m.notch_row <= ty0 + TY - 1;
}

__device__ __forceinline__ Slot tile_slot(const DMesh& m, const TileRows& R, int tx0, int ty0,
                                          int s) {
  Slot sl;
  if (s < HX * HY) {
    sl.hx = s % HX;
    sl.hy = s / HX;
    const int i = tx0 - 1 + sl.hx;
    sl.id = tile_node(R, sl.hy, i);
    sl.owned = sl.hx >= 1 && sl.hx <= TX && sl.hy >= 1 && sl.hy <= TY;
  } else {
    sl.hx = s - HX * HY;
    sl.hy = -1;
    const int i = tx0 - 1 + sl.hx;
    sl.id = is_dup_col(m, i) ? m.dup_start + (i - m.notch_lo) : -1;
    const bool row_owned = m.notch_row >= ty0 && m.notch_row < ty0 + TY;
    sl.owned = row_owned && sl.hx >= 1 && sl.hx <= TX;
  }
  return sl;
}

template <class T>
__device__ __forceinline__ void cell_corners(const DMesh& m, const T (&grid)[HY][HX],
                                             const T (&dup)[HX], int ex, int ey, int ci, int cj,
                                             T (&c)[4]) {
  c[0] = grid[ey][ex];
  c[1] = grid[ey][ex + 1];
  c[2] = grid[ey + 1][ex + 1];
  c[3] = grid[ey + 1][ex];
  if (cj == m.notch_row) {
    if (is_dup_col(m, ci)) c[0] = dup[ex];
    if (is_dup_col(m, ci + 1)) c[1] = dup[ex + 1];
  }
}

__device__ __forceinline__ double2 add2(double2 a, double2 b) {
  return make_double2(a.x + b.x, a.y + b.y);
}

// owned node (ox, oy): contributions of the cells below (corners 2, 3) and above (0, 1)
template <class T>
__device__ __forceinline__ void gather_corners(const T (&f)[4][EY][EX], int ox, int oy,
                                               T& below, T& above);
template <>
__device__ __forceinline__ void gather_corners<double2>(const double2 (&f)[4][EY][EX], int ox,
                                                        int oy, double2& below, double2& above) {
  below = add2(f[2][oy][ox], f[3][oy][ox + 1]);
  above = add2(f[0][oy + 1][ox + 1], f[1][oy + 1][ox]);
}
template <>
__device__ __forceinline__ void gather_corners<double>(const double (&f)[4][EY][EX], int ox,
                                                       int oy, double& below, double& above) {
  below = f[2][oy][ox] + f[3][oy][ox + 1];
  above = f[0][oy + 1][ox + 1] + f[1][oy + 1][ox];
}

__device__ __forceinline__ bool owned_split(const DMesh& m, int i, int j) {
  return j == m.notch_row && is_dup_col(m, i);
}

// ========================================================================================
// Momentum element ops
__device__ __forceinline__ void mom_cell_g(const Consts& C, const double (&dc)[4],
                                           double (&g)[4]) {
  double dg[4];
  interp_q4(C, dc[0], dc[1], dc[2], dc[3], dg);
#pragma unroll
  for (int q = 0; q < 4; ++q) g[q] = degradation(C, dg[q]);
}

// tangent apply K_e(u,d) p_e  (material.py:185-201, assembly.py:192-194)
__device__ __forceinline__ void mom_cell_apply(const Consts& C, const double2 (&pc)[4],
                                               const double (&g)[4], unsigned flags,
                                               double2 (&f)[4]) {
  Strain4 s;
  strain_q4(C, pc[0], pc[1], pc[2], pc[3], s);
  double sxx[4], syy[4], sxy[4];
#pragma unroll
  for (int q = 0; q < 4; ++q)
    tangent_gp(C, s.exx[q], s.eyy[q], s.gxy[q], g[q], (flags >> q) & 1u, sxx[q], syy[q], sxy[q]);
  backproject_q4(C, sxx, syy, sxy, f);
}

// ========================================================================================
// K1/K2/K3: momentum residual R = F_int(u, d), branch flags, Jacobi diagonal; CG init.
// One CTA per active tile.  partials[tile] = sum over free dofs of R^2.
struct MomPrepArgs {
  DMesh m;
  Consts C;
  const double2* u;
  const double* d;
  const uchar2* umask;
  double2* R;       // internal force (= residual, no external force on the hot path)
  double2* r;       // CG residual init: -R on free dofs, 0 on constrained
  double2* x;       // CG solution init: 0
  double2* dinv;    // masked inverse diagonal
  uint8_t* flags;   // [n_elems]
  double2* diag;    // optional raw diagonal (unmasked), may be null
  double* partials;
  int full;         // 0: residual only (R, partials)
};

__global__ void __launch_bounds__(NT) k_mom_prepare(MomPrepArgs a) {
  __shared__ SmemVec2Tile S;
  const DMesh& m = a.m;
  const Consts& C = a.C;
  const int2 t = m.tiles[blockIdx.x];
  const int tx0 = t.x * TX, ty0 = t.y * TY;
  load_tile_rows(m, ty0, S.R);
  __syncthreads();
  const bool dup = tile_has_dup(m, ty0);
  const int nslots = HX * HY + (dup ? HX : 0);
  for (int s = threadIdx.x; s < nslots; s += NT) {
    const Slot sl = tile_slot(m, S.R, tx0, ty0, s);
    double2 uv = make_double2(0.0, 0.0);
    double dv = 0.0;
    if (sl.id >= 0) {
      uv = ldro(a.u + sl.id);
      dv = ldro(a.d + sl.id);
    }
    if (sl.hy >= 0) { S.p[sl.hy][sl.hx] = uv; S.d[sl.hy][sl.hx] = dv; }
    else { S.pdup[sl.hx] = uv; S.ddup[sl.hx] = dv; }
  }
  __syncthreads();
  // pass 1: internal force + flags
  for (int c = threadIdx.x; c < EX * EY; c += NT) {
    const int ex = c % EX, ey = c / EX;
    const int ci = tx0 - 1 + ex, cj = ty0 - 1 + ey;
    const int eid = tile_cell(S.R, ey, ci);
    double2 f[4] = {{0, 0}, {0, 0}, {0, 0}, {0, 0}};
    if (eid >= 0) {
      double2 uc[4];
      double dc[4], g[4];
      cell_corners(m, S.p, S.pdup, ex, ey, ci, cj, uc);
      cell_corners(m, S.d, S.ddup, ex, ey, ci, cj, dc);
      mom_cell_g(C, dc, g);
      Strain4 st;
      strain_q4(C, uc[0], uc[1], uc[2], uc[3], st);
      double sxx[4], syy[4], sxy[4];
      unsigned fl = 0;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        bool plus;
        stress_gp(C, st.exx[q], st.eyy[q], st.gxy[q], g[q], sxx[q], syy[q], sxy[q], plus);
        fl |= (plus ? 1u : 0u) << q;
      }
      backproject_q4(C, sxx, syy, sxy, f);
      if (a.full && ex >= 1 && ey >= 1) a.flags[eid] = (uint8_t)fl;  // owner writes
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) S.f[q][ey][ex] = f[q];
  }
  __syncthreads();
  double rr = 0.0;
  double2 Rown[2];  // (orig, dup) residual of this thread's owned slot
  int idown[2] = {-1, -1};
  const int o = threadIdx.x;  // NT == TX*TY: one owned node per thread
  const int ox = o % TX, oy = o / TX;
  const int oi = tx0 + ox, oj = ty0 + oy;
  {
    const int id = tile_node(S.R, oy + 1, oi);
    if (id >= 0) {
      double2 below, above;
      gather_corners(S.f, ox, oy, below, above);
      if (owned_split(m, oi, oj)) {
        Rown[0] = below;
        Rown[1] = above;
        idown[0] = id;
        idown[1] = m.dup_start + (oi - m.notch_lo);
      } else {
        Rown[0] = add2(below, above);
        idown[0] = id;
      }
    }
  }
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    if (idown[k] < 0) continue;
    const int id = idown[k];
    const double2 Rv = Rown[k];
    a.R[id] = Rv;
    const uchar2 mk = a.umask[id];
    if (mk.x) rr += Rv.x * Rv.x;
    if (mk.y) rr += Rv.y * Rv.y;
    if (a.full) {
      a.r[id] = make_double2(mk.x ? -Rv.x : 0.0, mk.y ? -Rv.y : 0.0);
      a.x[id] = make_double2(0.0, 0.0);
    }
  }
  if (a.full) {
    __syncthreads();
    // pass 2: Jacobi diagonal of K_uu(u, d)
    for (int c = threadIdx.x; c < EX * EY; c += NT) {
      const int ex = c % EX, ey = c / EX;
      const int ci = tx0 - 1 + ex, cj = ty0 - 1 + ey;
      const int eid = tile_cell(S.R, ey, ci);
      double2 f[4] = {{0, 0}, {0, 0}, {0, 0}, {0, 0}};
      if (eid >= 0) {
        double2 uc[4];
        double dc[4], g[4];
        cell_corners(m, S.p, S.pdup, ex, ey, ci, cj, uc);
        cell_corners(m, S.d, S.ddup, ex, ey, ci, cj, dc);
        mom_cell_g(C, dc, g);
        Strain4 st;
        strain_q4(C, uc[0], uc[1], uc[2], uc[3], st);
        double lam[4], sh[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const bool plus = (st.exx[q] + st.eyy[q]) >= 0.0;
          const double kv = plus ? g[q] * C.k : C.k;
          lam[q] = g[q] * C.mu43 + kv;
          sh[q] = g[q] * C.mu;
        }
        diag_q4(C, lam, sh, f);
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) S.f[q][ey][ex] = f[q];
    }
    __syncthreads();
    if (idown[0] >= 0) {
      double2 below, above, dg[2];
      gather_corners(S.f, ox, oy, below, above);
      if (idown[1] >= 0) { dg[0] = below; dg[1] = above; }
      else dg[0] = add2(below, above);
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        if (idown[k] < 0) continue;
        const int id = idown[k];
        const uchar2 mk = a.umask[id];
        if (a.diag) a.diag[id] = dg[k];
        a.dinv[id] = make_double2(mk.x ? 1.0 / dg[k].x : 0.0, mk.y ? 1.0 / dg[k].y : 0.0);
      }
    }
  }
  double v[1] = {rr};
  block_sum<1>(v, S.red);
  if (threadIdx.x == 0) a.partials[blockIdx.x] = v[0];
}

// ========================================================================================
// K6/K7: phase-field residual R_d, Newton coefficient b (with optional fast-scheme extra
// stiffness on gated GPs), Jacobi diagonal, CG init.  partials[3*tile + {0,1,2}] =
// (sum free R^2, gated GP count, free nodes with non-positive diagonal).
struct EvoPrepArgs {
  DMesh m;
  Consts C;
  const double* d;
  const double* dprev;
  const double* psi;     // [n_elems*4]
  const double* trp;
  const double* dev2;
  const double* psimax;
  const uint8_t* pmask;
  double* R;
  double* r;
  double* x;
  double* dinv;
  double* b;             // [n_elems*4] Newton coefficient incl. extra
  double* diag;          // optional raw diagonal
  double* partials;
  int full;              // 0: residual only
  int extra_scheme;      // 0: none, 1..3: S1..S3 extra stiffness on gated GPs
};

__device__ __forceinline__ void load4(const double* p, int eid, double (&v)[4]) {
  const double2* q = reinterpret_cast<const double2*>(p + 4 * (size_t)eid);
  const double2 a = __ldg(q), b = __ldg(q + 1);
  v[0] = a.x; v[1] = a.y; v[2] = b.x; v[3] = b.y;
}
__device__ __forceinline__ void load4cg(const double* p, int eid, double (&v)[4]) {
  const double2* q = reinterpret_cast<const double2*>(p + 4 * (size_t)eid);
  const double2 a = __ldcg(q), b = __ldcg(q + 1);
  v[0] = a.x; v[1] = a.y; v[2] = b.x; v[3] = b.y;
}
__device__ __forceinline__ void store4(double* p, int eid, const double (&v)[4]) {
  double2* q = reinterpret_cast<double2*>(p + 4 * (size_t)eid);
  q[0] = make_double2(v[0], v[1]);
  q[1] = make_double2(v[2], v[3]);
}

__global__ void __launch_bounds__(NT) k_evo_prepare(EvoPrepArgs a) {
  __shared__ SmemScalTile S;
  const DMesh& m = a.m;
  const Consts& C = a.C;
  const int2 t = m.tiles[blockIdx.x];
  const int tx0 = t.x * TX, ty0 = t.y * TY;
  load_tile_rows(m, ty0, S.R);
  __syncthreads();
  const bool dup = tile_has_dup(m, ty0);
  const int nslots = HX * HY + (dup ? HX : 0);
  for (int s = threadIdx.x; s < nslots; s += NT) {
    const Slot sl = tile_slot(m, S.R, tx0, ty0, s);
    double dv = 0.0, pv = 0.0;
    if (sl.id >= 0) { dv = ldro(a.d + sl.id); pv = ldro(a.dprev + sl.id); }
    if (sl.hy >= 0) { S.p[sl.hy][sl.hx] = dv; S.a[sl.hy][sl.hx] = pv; }
    else { S.pdup[sl.hx] = dv; S.adup[sl.hx] = pv; }
  }
  __syncthreads();
  double ngate = 0.0;
  // pass 1: residual (assembly.py:217-228) and b (:233-239, schemes.py:112-142)
  for (int c = threadIdx.x; c < EX * EY; c += NT) {
    const int ex = c % EX, ey = c / EX;
    const int ci = tx0 - 1 + ex, cj = ty0 - 1 + ey;
    const int eid = tile_cell(S.R, ey, ci);
    double f[4] = {0, 0, 0, 0};
    if (eid >= 0) {
      double dc[4], pc[4], dg[4], pg[4], psi[4];
      cell_corners(m, S.p, S.pdup, ex, ey, ci, cj, dc);
      cell_corners(m, S.a, S.adup, ex, ey, ci, cj, pc);
      interp_q4(C, dc[0], dc[1], dc[2], dc[3], dg);
      interp_q4(C, pc[0], pc[1], pc[2], pc[3], pg);
      load4(a.psi, eid, psi);
      double aw[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const double x = dg[q] - pg[q];
        const double pen = C.gamma * (0.5 * (x - fabs(x)));
        const double src = C.at2 ? (C.src_base * 2.0) * dg[q] : C.src_base;
        aw[q] = (-2.0 * (1.0 - dg[q]) * psi[q] + src + pen) * C.w;
      }
#pragma unroll
      for (int aa = 0; aa < 4; ++aa) {
        double s = C.N[0][aa] * aw[0] + C.N[1][aa] * aw[1] + C.N[2][aa] * aw[2] +
                   C.N[3][aa] * aw[3];
        s += C.lap[aa][0] * dc[0] + C.lap[aa][1] * dc[1] + C.lap[aa][2] * dc[2] +
             C.lap[aa][3] * dc[3];
        f[aa] = s;
      }
      if (a.full && ex >= 1 && ey >= 1) {  // owner cell writes b
        double bq[4];
        const double srcd = C.at2 ? C.src_base * 2.0 : 0.0;
        double trp[4], dev2[4], pm[4];
        if (a.extra_scheme) {
          load4(a.trp, eid, trp);
          load4(a.dev2, eid, dev2);
          load4(a.psimax, eid, pm);
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          bq[q] = 2.0 * psi[q] + srcd + C.gamma * (dg[q] < pg[q] ? 1.0 : 0.0);
          if (a.extra_scheme && gate_gp(C, psi[q], pm[q], dg[q])) {
            bq[q] = bq[q] + extra_gp(C, a.extra_scheme, dg[q], trp[q], dev2[q]);
            ngate += 1.0;
          }
        }
        store4(a.b, eid, bq);
      }
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) S.f[q][ey][ex] = f[q];
  }
  __syncthreads();
  double rr = 0.0, nonpos = 0.0;
  const int o = threadIdx.x;
  const int ox = o % TX, oy = o / TX;
  const int oi = tx0 + ox, oj = ty0 + oy;
  double Rown[2];
  int idown[2] = {-1, -1};
  {
    const int id = tile_node(S.R, oy + 1, oi);
    if (id >= 0) {
      double below, above;
      gather_corners(S.f, ox, oy, below, above);
      if (owned_split(m, oi, oj)) {
        Rown[0] = below; Rown[1] = above;
        idown[0] = id; idown[1] = m.dup_start + (oi - m.notch_lo);
      } else {
        Rown[0] = below + above;
        idown[0] = id;
      }
    }
  }
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    if (idown[k] < 0) continue;
    const int id = idown[k];
    const double Rv = Rown[k];
    if (a.R) a.R[id] = Rv;
    const bool fr = a.pmask[id] != 0;
    if (fr) rr += Rv * Rv;
    if (a.full) {
      a.r[id] = fr ? -Rv : 0.0;
      a.x[id] = 0.0;
    }
  }
  if (a.full) {
    __syncthreads();
    // pass 2: diagonal sum_g N_a^2 b_g w + lap_aa (needs every b of the cell region: b of
    // non-owned cells is recomputed, not read, to avoid a cross-CTA dependency)
    for (int c = threadIdx.x; c < EX * EY; c += NT) {
      const int ex = c % EX, ey = c / EX;
      const int ci = tx0 - 1 + ex, cj = ty0 - 1 + ey;
      const int eid = tile_cell(S.R, ey, ci);
      double f[4] = {0, 0, 0, 0};
      if (eid >= 0) {
        double dc[4], pc[4], dg[4], pg[4], psi[4], bq[4];
        cell_corners(m, S.p, S.pdup, ex, ey, ci, cj, dc);
        cell_corners(m, S.a, S.adup, ex, ey, ci, cj, pc);
        interp_q4(C, dc[0], dc[1], dc[2], dc[3], dg);
        interp_q4(C, pc[0], pc[1], pc[2], pc[3], pg);
        load4(a.psi, eid, psi);
        const double srcd = C.at2 ? C.src_base * 2.0 : 0.0;
        double trp[4], dev2[4], pm[4];
        if (a.extra_scheme) {
          load4(a.trp, eid, trp);
          load4(a.dev2, eid, dev2);
          load4(a.psimax, eid, pm);
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          bq[q] = 2.0 * psi[q] + srcd + C.gamma * (dg[q] < pg[q] ? 1.0 : 0.0);
          if (a.extra_scheme && gate_gp(C, psi[q], pm[q], dg[q]))
            bq[q] = bq[q] + extra_gp(C, a.extra_scheme, dg[q], trp[q], dev2[q]);
        }
#pragma unroll
        for (int aa = 0; aa < 4; ++aa)
          f[aa] = C.Nw[0][aa] * C.N[0][aa] * bq[0] + C.Nw[1][aa] * C.N[1][aa] * bq[1] +
                  C.Nw[2][aa] * C.N[2][aa] * bq[2] + C.Nw[3][aa] * C.N[3][aa] * bq[3] +
                  C.lap[aa][aa];
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) S.f[q][ey][ex] = f[q];
    }
    __syncthreads();
    if (idown[0] >= 0) {
      double below, above, dg[2];
      gather_corners(S.f, ox, oy, below, above);
      if (idown[1] >= 0) { dg[0] = below; dg[1] = above; }
      else dg[0] = below + above;
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        if (idown[k] < 0) continue;
        const int id = idown[k];
        const bool fr = a.pmask[id] != 0;
        if (a.diag) a.diag[id] = dg[k];
        if (fr && !(dg[k] > 0.0)) nonpos += 1.0;
        a.dinv[id] = fr ? 1.0 / dg[k] : 0.0;
      }
    }
  }
  double v[3] = {rr, ngate, nonpos};
  block_sum<3>(v, S.red);
  if (threadIdx.x == 0) {
    a.partials[3 * blockIdx.x + 0] = v[0];
    a.partials[3 * blockIdx.x + 1] = v[1];
    a.partials[3 * blockIdx.x + 2] = v[2];
  }
}

// ========================================================================================
// K4/K8 + K5 (+K10): persistent Jacobi-PCG, one cooperative launch per linear solve.
// Mirrors scipy.sparse.linalg.cg (SciPy 1.18.1, called at linsolve.py:51): x0 = 0,
// stop when ||r|| < rtol*||b|| (recursive residual), z = D^-1 r, maxiter = 20 n.
// Per iteration, two grid barriers:
//   phase A (tiles): p_k = z + beta p_{k-1} evaluated on the fly for tile+halo nodes
//                    (p double-buffered), x += alpha_{k-1} p_{k-1} on owned nodes,
//                    q = A p_k (masked), partial p.q
//   phase B (flat):  r -= alpha q, partial r.r and r.D^-1.r
// The curvature probe (SPD predicate, SURVEY.md §7 hard part 1) aborts at p.q <= 0.
enum CgStatus { CG_CONVERGED = 0, CG_MAXITER = 1, CG_INDEFINITE = 2, CG_NAN = 3 };

struct CgResult {
  long long iters;
  int status;
  int pad;
  double bnorm, rnorm;
};

struct CgArgs {
  DMesh m;
  Consts C;
  int vec2;              // 1: momentum (double2 nodes), 0: phase field (double nodes)
  long long ndof;        // flat length (2*n_nodes or n_nodes)
  // momentum operator data
  const double* d;       // nodal d
  const uint8_t* flags;  // per element
  // phase-field operator data
  const double* b;       // [n_elems*4]
  // PCG vectors (flat doubles, length ndof)
  double* x;
  double* r;
  double* q;
  double* p0;
  double* p1;
  const double* dinv;
  double* target;        // optional: target += x at the end
  double* partials;      // >= 2*gridDim.x
  CgResult* result;
  double rtol;
  long long maxiter;
  int probe;             // abort on non-positive curvature
};

struct __align__(16) SmemCg {
  union {
    SmemVec2Tile v2;
    SmemScalTile s;
  };
  double bc[4];
};

// ---- phase A, momentum tile
__device__ __forceinline__ void cg_phaseA_mom(const CgArgs& a, SmemVec2Tile& S, int tile,
                                              bool first, double beta, double alpha_prev,
                                              const double2* __restrict__ pold,
                                              double2* __restrict__ pnew, double& pq) {
  const DMesh& m = a.m;
  const Consts& C = a.C;
  const int2 t = m.tiles[tile];
  const int tx0 = t.x * TX, ty0 = t.y * TY;
  load_tile_rows(m, ty0, S.R);
  __syncthreads();
  const bool dup = tile_has_dup(m, ty0);
  const int nslots = HX * HY + (dup ? HX : 0);
  const double2* r2 = reinterpret_cast<const double2*>(a.r);
  const double2* di2 = reinterpret_cast<const double2*>(a.dinv);
  double2* x2 = reinterpret_cast<double2*>(a.x);
  for (int s = threadIdx.x; s < nslots; s += NT) {
    const Slot sl = tile_slot(m, S.R, tx0, ty0, s);
    double2 pn = make_double2(0.0, 0.0);
    double dv = 0.0;
    if (sl.id >= 0) {
      const double2 rv = ldcg(r2 + sl.id);
      const double2 dv2 = ldro(di2 + sl.id);
      pn = make_double2(dv2.x * rv.x, dv2.y * rv.y);
      if (!first) {
        const double2 po = ldcg(pold + sl.id);
        pn.x = beta * po.x + pn.x;
        pn.y = beta * po.y + pn.y;
        if (sl.owned) {
          double2 xv = ldcg(x2 + sl.id);
          xv.x += alpha_prev * po.x;
          xv.y += alpha_prev * po.y;
          x2[sl.id] = xv;
        }
      }
      if (sl.owned) pnew[sl.id] = pn;
      dv = ldro(a.d + sl.id);
    }
    if (sl.hy >= 0) { S.p[sl.hy][sl.hx] = pn; S.d[sl.hy][sl.hx] = dv; }
    else { S.pdup[sl.hx] = pn; S.ddup[sl.hx] = dv; }
  }
  __syncthreads();
  for (int c = threadIdx.x; c < EX * EY; c += NT) {
    const int ex = c % EX, ey = c / EX;
    const int ci = tx0 - 1 + ex, cj = ty0 - 1 + ey;
    const int eid = tile_cell(S.R, ey, ci);
    double2 f[4] = {{0, 0}, {0, 0}, {0, 0}, {0, 0}};
    if (eid >= 0) {
      double2 pc[4];
      double dc[4], g[4];
      cell_corners(m, S.p, S.pdup, ex, ey, ci, cj, pc);
      cell_corners(m, S.d, S.ddup, ex, ey, ci, cj, dc);
      mom_cell_g(C, dc, g);
      mom_cell_apply(C, pc, g, __ldg(a.flags + eid), f);
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) S.f[q][ey][ex] = f[q];
  }
  __syncthreads();
  double2* q2 = reinterpret_cast<double2*>(a.q);
  {
    const int o = threadIdx.x;
    const int ox = o % TX, oy = o / TX;
    const int oi = tx0 + ox, oj = ty0 + oy;
    const int id = tile_node(S.R, oy + 1, oi);
    if (id >= 0) {
      double2 below, above;
      gather_corners(S.f, ox, oy, below, above);
      const bool split = owned_split(m, oi, oj);
      double2 qv = split ? below : add2(below, above);
      double2 dv = ldro(di2 + id);
      qv.x = dv.x != 0.0 ? qv.x : 0.0;
      qv.y = dv.y != 0.0 ? qv.y : 0.0;
      q2[id] = qv;
      const double2 pv = S.p[oy + 1][ox + 1];
      pq += pv.x * qv.x + pv.y * qv.y;
      if (split) {
        const int idd = m.dup_start + (oi - m.notch_lo);
        double2 qd = above;
        dv = ldro(di2 + idd);
        qd.x = dv.x != 0.0 ? qd.x : 0.0;
        qd.y = dv.y != 0.0 ? qd.y : 0.0;
        q2[idd] = qd;
        const double2 pd = S.pdup[ox + 1];
        pq += pd.x * qd.x + pd.y * qd.y;
      }
    }
  }
  __syncthreads();
}

// ---- phase A, phase-field tile
__device__ __forceinline__ void cg_phaseA_evo(const CgArgs& a, SmemScalTile& S, int tile,
                                              bool first, double beta, double alpha_prev,
                                              const double* __restrict__ pold,
                                              double* __restrict__ pnew, double& pq) {
  const DMesh& m = a.m;
  const Consts& C = a.C;
  const int2 t = m.tiles[tile];
  const int tx0 = t.x * TX, ty0 = t.y * TY;
  load_tile_rows(m, ty0, S.R);
  __syncthreads();
  const bool dup = tile_has_dup(m, ty0);
  const int nslots = HX * HY + (dup ? HX : 0);
  for (int s = threadIdx.x; s < nslots; s += NT) {
    const Slot sl = tile_slot(m, S.R, tx0, ty0, s);
    double pn = 0.0;
    if (sl.id >= 0) {
      pn = ldro(a.dinv + sl.id) * ldcg(a.r + sl.id);
      if (!first) {
        const double po = ldcg(pold + sl.id);
        pn = beta * po + pn;
        if (sl.owned) a.x[sl.id] = ldcg(a.x + sl.id) + alpha_prev * po;
      }
      if (sl.owned) pnew[sl.id] = pn;
    }
    if (sl.hy >= 0) S.p[sl.hy][sl.hx] = pn;
    else S.pdup[sl.hx] = pn;
  }
  __syncthreads();
  for (int c = threadIdx.x; c < EX * EY; c += NT) {
    const int ex = c % EX, ey = c / EX;
    const int ci = tx0 - 1 + ex, cj = ty0 - 1 + ey;
    const int eid = tile_cell(S.R, ey, ci);
    double f[4] = {0, 0, 0, 0};
    if (eid >= 0) {
      double pc[4], pg[4], bq[4];
      cell_corners(m, S.p, S.pdup, ex, ey, ci, cj, pc);
      interp_q4(C, pc[0], pc[1], pc[2], pc[3], pg);
      load4(a.b, eid, bq);
      double t4[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) t4[q] = bq[q] * pg[q];
#pragma unroll
      for (int aa = 0; aa < 4; ++aa)
        f[aa] = C.Nw[0][aa] * t4[0] + C.Nw[1][aa] * t4[1] + C.Nw[2][aa] * t4[2] +
                C.Nw[3][aa] * t4[3] + C.lap[aa][0] * pc[0] + C.lap[aa][1] * pc[1] +
                C.lap[aa][2] * pc[2] + C.lap[aa][3] * pc[3];
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) S.f[q][ey][ex] = f[q];
  }
  __syncthreads();
  {
    const int o = threadIdx.x;
    const int ox = o % TX, oy = o / TX;
    const int oi = tx0 + ox, oj = ty0 + oy;
    const int id = tile_node(S.R, oy + 1, oi);
    if (id >= 0) {
      double below, above;
      gather_corners(S.f, ox, oy, below, above);
      const bool split = owned_split(m, oi, oj);
      double qv = split ? below : below + above;
      qv = ldro(a.dinv + id) != 0.0 ? qv : 0.0;
      a.q[id] = qv;
      pq += S.p[oy + 1][ox + 1] * qv;
      if (split) {
        const int idd = m.dup_start + (oi - m.notch_lo);
        const double qd = ldro(a.dinv + idd) != 0.0 ? above : 0.0;
        a.q[idd] = qd;
        pq += S.pdup[ox + 1] * qd;
      }
    }
  }
  __syncthreads();
}

// grid-wide deterministic reduction of NV partials per CTA (called right after grid.sync)
// partial k of CTA i lives at part[stride*i + k]
template <int NV>
__device__ __forceinline__ void grid_reduce(const double* part, int stride, double* bc,
                                            double (&out)[NV]) {
  if (threadIdx.x < 32) {
    double s[NV];
#pragma unroll
    for (int k = 0; k < NV; ++k) s[k] = 0.0;
    for (int i = threadIdx.x; i < (int)gridDim.x; i += 32) {
#pragma unroll
      for (int k = 0; k < NV; ++k) s[k] += __ldcg(part + stride * i + k);
    }
#pragma unroll
    for (int k = 0; k < NV; ++k) s[k] = warp_sum(s[k]);
    if (threadIdx.x == 0) {
#pragma unroll
      for (int k = 0; k < NV; ++k) bc[k] = s[k];
    }
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < NV; ++k) out[k] = bc[k];
}

// flat pass: r -= alpha q (alpha = 0 for the initial reduction); partials (r.r, r.Dinv.r)
__device__ __forceinline__ void cg_phaseB(const CgArgs& a, double alpha, bool update,
                                          double& rr, double& rz) {
  const long long n2 = a.ndof >> 1;
  const long long stride = (long long)gridDim.x * blockDim.x;
  double2* r2 = reinterpret_cast<double2*>(a.r);
  const double2* q2 = reinterpret_cast<const double2*>(a.q);
  const double2* d2 = reinterpret_cast<const double2*>(a.dinv);
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n2; i += stride) {
    double2 rv = ldcg(r2 + i);
    if (update) {
      const double2 qv = ldcg(q2 + i);
      rv.x -= alpha * qv.x;
      rv.y -= alpha * qv.y;
      r2[i] = rv;
    }
    const double2 dv = ldro(d2 + i);
    rr += rv.x * rv.x + rv.y * rv.y;
    rz += rv.x * (dv.x * rv.x) + rv.y * (dv.y * rv.y);
  }
  if ((a.ndof & 1) && blockIdx.x == 0 && threadIdx.x == 0) {
    const long long i = a.ndof - 1;
    double rv = __ldcg(a.r + i);
    if (update) {
      rv -= alpha * __ldcg(a.q + i);
      a.r[i] = rv;
    }
    rr += rv * rv;
    rz += rv * (__ldg(a.dinv + i) * rv);
  }
}

__global__ void __launch_bounds__(NT) k_cg(CgArgs a) {
  __shared__ SmemCg S;
  cg::grid_group grid = cg::this_grid();
  double* part = a.partials;
  // initial reduction: ||b||^2 and b.D^-1.b (r = b on entry)
  double rr = 0.0, rz = 0.0;
  cg_phaseB(a, 0.0, false, rr, rz);
  {
    double v[2] = {rr, rz};
    block_sum<2>(v, a.vec2 ? S.v2.red : S.s.red);
    if (threadIdx.x == 0) { part[2 * blockIdx.x] = v[0]; part[2 * blockIdx.x + 1] = v[1]; }
  }
  grid.sync();
  double red[2];
  grid_reduce<2>(part, 2, S.bc, red);
  rr = red[0];
  double rho = red[1];
  const double bnorm = sqrt(rr);
  const double atol = a.rtol * bnorm;
  long long k = 0;
  int status = CG_CONVERGED;
  double alpha = 0.0, rho_prev = 0.0;
  if (bnorm != 0.0) {
    for (;;) {
      const double rn = sqrt(rr);
      if (rn < atol) break;
      if (!(rn == rn)) { status = CG_NAN; break; }
      if (k >= a.maxiter) { status = CG_MAXITER; break; }
      const bool first = (k == 0);
      const double beta = first ? 0.0 : rho / rho_prev;
      double* pnew = (k & 1) ? a.p1 : a.p0;
      const double* pold = (k & 1) ? a.p0 : a.p1;
      double pq = 0.0;
      for (int tile = blockIdx.x; tile < a.m.n_tiles; tile += gridDim.x) {
        if (a.vec2)
          cg_phaseA_mom(a, S.v2, tile, first, beta, alpha,
                        reinterpret_cast<const double2*>(pold),
                        reinterpret_cast<double2*>(pnew), pq);
        else
          cg_phaseA_evo(a, S.s, tile, first, beta, alpha, pold, pnew, pq);
      }
      {
        double v[1] = {pq};
        block_sum<1>(v, a.vec2 ? S.v2.red : S.s.red);
        if (threadIdx.x == 0) part[2 * blockIdx.x] = v[0];
      }
      grid.sync();
      double pqr[1];
      grid_reduce<1>(part, 2, S.bc, pqr);
      const double pqv = pqr[0];
      if (a.probe && !(pqv > 0.0)) { status = CG_INDEFINITE; k += 1; break; }
      alpha = rho / pqv;
      rho_prev = rho;
      rr = 0.0; rz = 0.0;
      cg_phaseB(a, alpha, true, rr, rz);
      {
        double v[2] = {rr, rz};
        block_sum<2>(v, a.vec2 ? S.v2.red : S.s.red);
        if (threadIdx.x == 0) { part[2 * blockIdx.x] = v[0]; part[2 * blockIdx.x + 1] = v[1]; }
      }
      grid.sync();
      grid_reduce<2>(part, 2, S.bc, red);
      rr = red[0];
      rho = red[1];
      ++k;
    }
  }
  // finalize: x += alpha_{k-1} p_{k-1}; target += x
  if (status != CG_INDEFINITE) {
    const double* plast = (k & 1) ? a.p0 : a.p1;  // p_{k-1} lives in buffer (k-1)&1
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < a.ndof;
         i += stride) {
      double xv = __ldcg(a.x + i);
      if (k > 0) xv += alpha * __ldcg(plast + i);
      a.x[i] = xv;
      if (a.target) a.target[i] += xv;
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    a.result->iters = k;
    a.result->status = status;
    a.result->bnorm = bnorm;
    a.result->rnorm = sqrt(rr);
  }
}

// ========================================================================================
// matrix-free tangent apply (tests / pf_*_tangent_apply): y = K x, unmasked, at current state
struct ApplyArgs {
  DMesh m;
  Consts C;
  const double* d;       // momentum: nodal d
  const uint8_t* flags;  // momentum: branch flags
  const double* b;       // phase field: Newton coefficient
  const double* x;
  double* y;
  int vec2;
};

__global__ void __launch_bounds__(NT) k_apply(ApplyArgs a) {
  __shared__ SmemCg S;
  const DMesh& m = a.m;
  const Consts& C = a.C;
  const int2 t = m.tiles[blockIdx.x];
  const int tx0 = t.x * TX, ty0 = t.y * TY;
  TileRows& R = a.vec2 ? S.v2.R : S.s.R;
  load_tile_rows(m, ty0, R);
  __syncthreads();
  const bool dup = tile_has_dup(m, ty0);
  const int nslots = HX * HY + (dup ? HX : 0);
  for (int s = threadIdx.x; s < nslots; s += NT) {
    const Slot sl = tile_slot(m, R, tx0, ty0, s);
    if (a.vec2) {
      double2 pv = make_double2(0, 0);
      double dv = 0.0;
      if (sl.id >= 0) {
        pv = ldro(reinterpret_cast<const double2*>(a.x) + sl.id);
        dv = ldro(a.d + sl.id);
      }
      if (sl.hy >= 0) { S.v2.p[sl.hy][sl.hx] = pv; S.v2.d[sl.hy][sl.hx] = dv; }
      else { S.v2.pdup[sl.hx] = pv; S.v2.ddup[sl.hx] = dv; }
    } else {
      const double pv = sl.id >= 0 ? ldro(a.x + sl.id) : 0.0;
      if (sl.hy >= 0) S.s.p[sl.hy][sl.hx] = pv;
      else S.s.pdup[sl.hx] = pv;
    }
  }
  __syncthreads();
  for (int c = threadIdx.x; c < EX * EY; c += NT) {
    const int ex = c % EX, ey = c / EX;
    const int ci = tx0 - 1 + ex, cj = ty0 - 1 + ey;
    const int eid = tile_cell(R, ey, ci);
    if (a.vec2) {
      double2 f[4] = {{0, 0}, {0, 0}, {0, 0}, {0, 0}};
      if (eid >= 0) {
        double2 pc[4];
        double dc[4], g[4];
        cell_corners(m, S.v2.p, S.v2.pdup, ex, ey, ci, cj, pc);
        cell_corners(m, S.v2.d, S.v2.ddup, ex, ey, ci, cj, dc);
        mom_cell_g(C, dc, g);
        mom_cell_apply(C, pc, g, __ldg(a.flags + eid), f);
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) S.v2.f[q][ey][ex] = f[q];
    } else {
      double f[4] = {0, 0, 0, 0};
      if (eid >= 0) {
        double pc[4], pg[4], bq[4], t4[4];
        cell_corners(m, S.s.p, S.s.pdup, ex, ey, ci, cj, pc);
        interp_q4(C, pc[0], pc[1], pc[2], pc[3], pg);
        load4(a.b, eid, bq);
#pragma unroll
        for (int q = 0; q < 4; ++q) t4[q] = bq[q] * pg[q];
#pragma unroll
        for (int aa = 0; aa < 4; ++aa)
          f[aa] = C.Nw[0][aa] * t4[0] + C.Nw[1][aa] * t4[1] + C.Nw[2][aa] * t4[2] +
                  C.Nw[3][aa] * t4[3] + C.lap[aa][0] * pc[0] + C.lap[aa][1] * pc[1] +
                  C.lap[aa][2] * pc[2] + C.lap[aa][3] * pc[3];
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) S.s.f[q][ey][ex] = f[q];
    }
  }
  __syncthreads();
  const int o = threadIdx.x;
  const int ox = o % TX, oy = o / TX;
  const int oi = tx0 + ox, oj = ty0 + oy;
  const int id = tile_node(R, oy + 1, oi);
  if (id < 0) return;
  const bool split = owned_split(m, oi, oj);
  const int idd = split ? m.dup_start + (oi - m.notch_lo) : -1;
  if (a.vec2) {
    double2 below, above;
    gather_corners(S.v2.f, ox, oy, below, above);
    double2* y2 = reinterpret_cast<double2*>(a.y);
    y2[id] = split ? below : add2(below, above);
    if (split) y2[idd] = above;
  } else {
    double below, above;
    gather_corners(S.s.f, ox, oy, below, above);
    a.y[id] = split ? below : below + above;
    if (split) a.y[idd] = above;
  }
}

// ========================================================================================
// cell-parallel GP kernels (2-D grid over the bounding cell grid)
struct GpArgs {
  DMesh m;
  Consts C;
  const double2* u;
  const double* d;
  const double* dd;      // nodal damage increment (energy update)
  double* trp;
  double* dev2;
  double* psi;
  const double* psimax;
  double* strain;        // optional [n_elems*16]
  double* tr;            // optional [n_elems*4]
  uint8_t* gate;         // optional [n_elems*4]
  double* extra;         // optional [n_elems*4]
  int scheme;
};

// K1 / A8: refresh_gp_from_displacement (assembly.py:260-269)
__global__ void k_refresh_gp(GpArgs a) {
  const int ci = blockIdx.x * blockDim.x + threadIdx.x, cj = blockIdx.y;
  const int eid = cell_at(a.m, ci, cj);
  if (eid < 0) return;
  int n[4];
  cell_nodes(a.m, ci, cj, n);
  Strain4 s;
  strain_q4(a.C, ldro(a.u + n[0]), ldro(a.u + n[1]), ldro(a.u + n[2]), ldro(a.u + n[3]), s);
  double trv[4], trp[4], dev2[4], psi[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) invariants_gp(a.C, s.exx[q], s.eyy[q], s.gxy[q], trv[q], trp[q],
                                            dev2[q], psi[q]);
  if (a.trp) store4(a.trp, eid, trp);
  if (a.dev2) store4(a.dev2, eid, dev2);
  if (a.psi) store4(a.psi, eid, psi);
  if (a.tr) store4(a.tr, eid, trv);
  if (a.strain) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      double* e = a.strain + 16 * (size_t)eid + 4 * q;
      e[0] = s.exx[q]; e[1] = s.eyy[q]; e[2] = 0.0; e[3] = s.gxy[q];
    }
  }
}

// K9: update_active_energy (schemes.py:145-176) at GPs gated before the solve
// (gate recomputed from the unchanged pre-solve d, psi+, psi_max).
__global__ void k_update_energy(GpArgs a) {
  const int ci = blockIdx.x * blockDim.x + threadIdx.x, cj = blockIdx.y;
  const int eid = cell_at(a.m, ci, cj);
  if (eid < 0) return;
  int n[4];
  cell_nodes(a.m, ci, cj, n);
  double dg[4], ddg[4];
  interp_q4(a.C, ldro(a.d + n[0]), ldro(a.d + n[1]), ldro(a.d + n[2]), ldro(a.d + n[3]), dg);
  interp_q4(a.C, ldro(a.dd + n[0]), ldro(a.dd + n[1]), ldro(a.dd + n[2]), ldro(a.dd + n[3]),
            ddg);
  double trp[4], dev2[4], psi[4], pm[4];
  load4(a.trp, eid, trp);
  load4(a.dev2, eid, dev2);
  load4(a.psi, eid, psi);
  load4(a.psimax, eid, pm);
  bool any = false;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    if (!(gate_gp(a.C, psi[q], pm[q], dg[q]) && ddg[q] > 0.0)) continue;
    any = true;
    const double g = degradation(a.C, dg[q]);
    const double ratio = (1.0 - dg[q]) / g;
    const double y = 2.0 * ratio * ddg[q];
    if (a.scheme == 1 || a.scheme == 3) trp[q] = trp[q] * (1.0 + y);
    if (a.scheme == 2 || a.scheme == 3)
      dev2[q] = dev2[q] * (1.0 + 4.0 * (ratio * ddg[q] + ratio * ratio * (ddg[q] * ddg[q])));
    psi[q] = a.C.mu * dev2[q] + 0.5 * a.C.k * (trp[q] * trp[q]);
  }
  if (any) {
    store4(a.trp, eid, trp);
    store4(a.dev2, eid, dev2);
    store4(a.psi, eid, psi);
  }
}

// softening gate and extra stiffness (tests / pf_softening_gate, pf_extra_stiffness)
__global__ void k_gate_extra(GpArgs a) {
  const int ci = blockIdx.x * blockDim.x + threadIdx.x, cj = blockIdx.y;
  const int eid = cell_at(a.m, ci, cj);
  if (eid < 0) return;
  int n[4];
  cell_nodes(a.m, ci, cj, n);
  double dg[4], trp[4], dev2[4], psi[4], pm[4];
  interp_q4(a.C, ldro(a.d + n[0]), ldro(a.d + n[1]), ldro(a.d + n[2]), ldro(a.d + n[3]), dg);
  load4(a.trp, eid, trp);
  load4(a.dev2, eid, dev2);
  load4(a.psi, eid, psi);
  load4(a.psimax, eid, pm);
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const bool gt = gate_gp(a.C, psi[q], pm[q], dg[q]);
    if (a.gate) a.gate[4 * (size_t)eid + q] = gt ? 1 : 0;
    if (a.extra)
      a.extra[4 * (size_t)eid + q] =
          (gt && a.scheme) ? extra_gp(a.C, a.scheme, dg[q], trp[q], dev2[q]) : 0.0;
  }
}

// ========================================================================================
// small flat kernels
__global__ void k_add_inc(double* u, const long long* dofs, long long n, double inc) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) u[dofs[i]] += inc;
}

__global__ void k_axpy(double* y, const double* x, long long n) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) y[i] += x[i];
}

// K11: psi_max = max(psi_max, psi_plus); d_prev = d   (schemes.py:390-391)
__global__ void k_commit(double* psimax, const double* psi, long long ngp, double* dprev,
                         const double* d, long long nn) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < ngp) psimax[i] = fmax(psimax[i], psi[i]);
  if (i < nn) dprev[i] = d[i];
}

// fixed-order sum of nv interleaved partial streams -> out[k]
__global__ void k_finalize(const double* part, int n, int nv, double* out) {
  __shared__ double red[32 * 4];
  double s[4] = {0, 0, 0, 0};
  for (int i = threadIdx.x; i < n; i += blockDim.x)
    for (int k = 0; k < nv; ++k) s[k] += part[(size_t)nv * i + k];
  block_sum<4>(s, red);
  if (threadIdx.x == 0)
    for (int k = 0; k < nv; ++k) out[k] = s[k];
}

// A16: reaction force = sum over node set of F_int component (assembly.py:315-326)
__global__ void k_reaction(const double* R, const long long* nodes, long long n, int comp,
                           double* out) {
  __shared__ double red[32];
  double s[1] = {0.0};
  for (long long i = threadIdx.x; i < n; i += blockDim.x) s[0] += R[2 * nodes[i] + comp];
  block_sum<1>(s, red);
  if (threadIdx.x == 0) out[0] = s[0];
}

__global__ void k_flush(double* buf, long long n, double v) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    buf[i] = v;
}

}  // namespace pfb
