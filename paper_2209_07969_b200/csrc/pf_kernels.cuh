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

// Owned node (ox, oy) sums its (up to four) cell contributions SEQUENTIALLY in the reference's
// element order -- (i-1,j-1) corner 2, (i,j-1) corner 3, (i-1,j) corner 1, (i,j) corner 0 --
// i.e. exactly the accumulation order of np.add.at / COO->CSR duplicate summation
// (assembly.py:188, :195-197).  The order matters beyond round-off: the symmetric tension test
// bifurcates at the crack step and the side the crack takes is decided by this bias.
// `below` = first two terms (cells of row j-1), `above` = last two (cells of row j), used
// separately at slit nodes, which belong to one side only.
template <class T>
__device__ __forceinline__ T add_t(T a, T b);
template <>
__device__ __forceinline__ double add_t<double>(double a, double b) { return a + b; }
template <>
__device__ __forceinline__ double2 add_t<double2>(double2 a, double2 b) { return add2(a, b); }

template <class T>
__device__ __forceinline__ void gather_corners(const T (&f)[4][EY][EX], int ox, int oy,
                                               T& below, T& above) {
  below = add_t(f[2][oy][ox], f[3][oy][ox + 1]);
  above = add_t(f[1][oy + 1][ox], f[0][oy + 1][ox + 1]);
}
template <class T>
__device__ __forceinline__ T gather_all(const T (&f)[4][EY][EX], int ox, int oy) {
  return add_t(add_t(add_t(f[2][oy][ox], f[3][oy][ox + 1]), f[1][oy + 1][ox]),
               f[0][oy + 1][ox + 1]);
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
        Rown[0] = gather_all(S.f, ox, oy);
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
    if (node_owned(m, id)) {
      if (mk.x) rr += Rv.x * Rv.x;
      if (mk.y) rr += Rv.y * Rv.y;
    }
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
      else dg[0] = gather_all(S.f, ox, oy);
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
            if (cell_owned(m, eid)) ngate += 1.0;
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
        Rown[0] = gather_all(S.f, ox, oy);
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
    if (fr && node_owned(m, id)) rr += Rv * Rv;
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
      else dg[0] = gather_all(S.f, ox, oy);
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        if (idown[k] < 0) continue;
        const int id = idown[k];
        const bool fr = a.pmask[id] != 0;
        if (a.diag) a.diag[id] = dg[k];
        if (fr && !(dg[k] > 0.0) && node_owned(m, id)) nonpos += 1.0;
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

}  // namespace pfb
#include "pf_cg.cuh"
namespace pfb {

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

// interp_nodal (assembly.py:148-150): a nodal scalar field at the four Gauss points of each cell
__global__ void k_interp_nodal(GpArgs a, const double* __restrict__ field,
                               double* __restrict__ out) {
  const int ci = blockIdx.x * blockDim.x + threadIdx.x, cj = blockIdx.y;
  const int eid = cell_at(a.m, ci, cj);
  if (eid < 0) return;
  int n[4];
  cell_nodes(a.m, ci, cj, n);
  double v[4];
  interp_q4(a.C, ldro(field + n[0]), ldro(field + n[1]), ldro(field + n[2]), ldro(field + n[3]), v);
  store4(out, eid, v);
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

// Device-side pre-crack initialiser (configs.precrack_nodes): d = d_prev = 1
// at every node within `radius` of one of the segments (ax, ay, bx, by).  Node (i, j) sits at
// (i hx, j hy) like np.linspace(0, side, n + 1), the last column / row exactly at x_last /
// y_last; a slit position marks both crack faces (the base node and its duplicate share the
// coordinates).  The distance is the host's expression in the same operation order, without FMA
// contraction.
__global__ void k_precrack(DMesh m, double hx, double hy, double x_last, double y_last,
                           const double4* __restrict__ seg, int n_seg, double radius,
                           double* __restrict__ d, double* __restrict__ dprev) {
  const long long total = (long long)(m.nx + 1) * (m.ny + 1);
  for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(t % (m.nx + 1)), j = (int)(t / (m.nx + 1));
    const int4 rw = __ldg(m.nrow + j);
    if (i < rw.x || i >= rw.y) continue;
    const bool dpos = j == m.notch_row && i >= m.notch_lo && i < m.notch_hi;
    const int id = rw.z + (i - rw.x);
    const double px = i == m.nx ? x_last : __dmul_rn((double)i, hx);
    const double py = j == m.ny ? y_last : __dmul_rn((double)j, hy);
    bool hit = false;
    for (int k = 0; k < n_seg && !hit; ++k) {
      const double4 sg = seg[k];
      const double ex = __dsub_rn(sg.z, sg.x), ey = __dsub_rn(sg.w, sg.y);
      double tt = __ddiv_rn(__dadd_rn(__dmul_rn(__dsub_rn(px, sg.x), ex),
                                      __dmul_rn(__dsub_rn(py, sg.y), ey)),
                            __dadd_rn(__dmul_rn(ex, ex), __dmul_rn(ey, ey)));
      tt = fmin(fmax(tt, 0.0), 1.0);
      const double qx = __dsub_rn(px, __dadd_rn(sg.x, __dmul_rn(tt, ex)));
      const double qy = __dsub_rn(py, __dadd_rn(sg.y, __dmul_rn(tt, ey)));
      hit = hypot(qx, qy) <= radius;
    }
    if (hit) {
      d[id] = 1.0;
      dprev[id] = 1.0;
      if (dpos) {
        const int dup = m.dup_start + (i - m.notch_lo);
        d[dup] = 1.0;
        dprev[dup] = 1.0;
      }
    }
  }
}

__global__ void k_flush(double* buf, long long n, double v) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    buf[i] = v;
}

}  // namespace pfb
#include "pf_mg.cuh"
#include "pf_mgs.cuh"
#include "pf_mgd.cuh"
#include "pf_st.cuh"
