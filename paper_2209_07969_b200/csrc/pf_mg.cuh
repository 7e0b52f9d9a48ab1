// pf_mg.cuh — geometric-multigrid-preconditioned CG for the momentum systems (K4+K5 with a
// V-cycle preconditioner), executed as a CUDA graph whose PCG loop is a device-driven WHILE
// conditional node (no host round trip per iteration or per solve).
//
// Same linear system and stopping test as the reference's Jacobi-PCG switch (linsolve.py:48-54,
// SciPy 1.18.1 cg: x0 = 0, stop at the top of an iteration when the recursive residual satisfies
// ||r|| < rtol*||b||, maxiter = 20 n).  Only the preconditioner differs: M^-1 = one symmetric
// V(1,1)-cycle instead of D^-1, which cuts the iteration count from O(n_x) (~4000 at 512^2) to
// a few tens, independent of the mesh size.  Any SPD preconditioner gives the same solution to
// the same relative residual, so the Newton/staggered iteration counts are unchanged.
//
// Hierarchy (rebuilt at each solve; the tangent changes every Newton iteration):
//   * level 0 is the matrix-free fine operator (K_uu(u, d) of material.py:185-201 on the
//     reference's Q4 cells, masked at the Dirichlet dofs: assembly.py:279-312);
//   * level l+1 = 2x2 agglomeration of level l's cells (row-compact layout kept: L-panel rows,
//     the slit duplicated on every level) with bilinear prolongation P_l masked at dead dofs;
//   * Galerkin operators A_{l+1} = P^T A_l P, computed cell by cell: for nested Q4 cells the
//     restriction of P to one child cell is the parent's bilinear interpolation Q_c, so the
//     coarse cell matrix is K_E = sum_c Q_c^T K_c Q_c (exactly the global product; verified
//     against scipy in scripts/mg_study.py to 1e-16);
//   * smoother: one damped-Jacobi sweep before and after (omega_l = 4 / (3 lambda_l),
//     lambda_l = lambda_max(D_l^-1 A_l) from MG_POW power steps in the setup);
//   * coarsest level: dense inverse (<= MG_DENSE_MAX dofs) or nu_c Jacobi sweeps.
// Kernels: the fine level is a warp march over its cells (mg_march: the barrier-free register
// march of pf_march.cuh, generic in the node input/output functors), the coarse levels are node
// gathers over their stored cell matrices, and the smallest levels ("tail") run as one
// single-CTA kernel with CTA barriers.  Reductions are per-CTA partials summed in a fixed order
// (last-block pattern), so every result is bit-reproducible run to run.
#pragma once

namespace pfb {

constexpr int MG_MAXL = 14;
constexpr int MG_NT = 256;
constexpr int MG_WARPS = MG_NT / 32;
constexpr int MG_POW = 8;          // power steps for lambda_max(D^-1 A_l)
constexpr int MG_DENSE_MAX = 64;   // coarsest level by a dense inverse when 2 n_nodes <= this
constexpr int MG_TAIL_NT = 512;    // threads of the single-CTA tail kernel

struct MgLevel {
  DMesh m;        // row tables (nrow/erow), notch, n_nodes/n_elems of this level
  double* K;      // [n_elems][64] Galerkin cell matrices (l >= 1)
  double* dinv;   // [2 n_nodes] inverse diagonal (0 = constrained / dead dof)
  double* b;      // right-hand side (l >= 1)
  double* t;      // residual / prolongated iterate / power-iteration buffer
  double* e;      // correction / power-iteration buffer
  int items;      // node items (rows x 32-column chunks) of mg_for_nodes
  int item_off;   // offset of this level in the concatenated coarse item space (power steps)
};

// device-side control block of one solve
struct MgIn {  // per-solve inputs, in mapped pinned host memory (read by k_mg_init)
  double rtol;
  long long maxiter;
  double* target;  // optional: target += x at the end
};
struct MgCtl {
  double omega[MG_MAXL];
  double* target;
  double rho_prev, bnorm, atol, rr;
  long long k, maxiter;
  int status, done;
  unsigned int count;  // last-block counter (reset by the last block)
};

struct MgArgs {
  Consts C;
  int n_levels, n_tail;  // levels [1, n_tail) by grid kernels, [n_tail, n_levels) by k_mg_tail
  int dense, nu_c;
  MgLevel L[MG_MAXL];
  MarchGeom g0;          // march units of the fine level
  int coarse_items;      // sum of items over levels >= 1
  const double* d;       // nodal d (level-0 operator)
  const uint8_t* flags;  // level-0 tangent branch bits
  double *x, *r, *z, *p0, *p1, *q;
  double* Ainv;          // [nd*nd] dense inverse of the coarsest level
  double* part;          // per-CTA partial sums (>= max grid * 2 * MG_MAXL)
  MgCtl* ctl;
  const MgIn* in;
  CgResult* result;
  long long ndof;
  cudaGraphConditionalHandle cond;
  int use_cond;          // 0: launched outside the graph (per-kernel profiling)
};

struct MgWarp {
  int4 nwin[32], ewin[32];
  double2 dv[32];
  double da[32];
  int did[32];
};
struct MgGal {
  double Kc[4][64];
  double T[4][64];
};

__device__ __forceinline__ double2 d2add(double2 a, double2 b) {
  return make_double2(a.x + b.x, a.y + b.y);
}
__device__ __forceinline__ double2 d2ldcg(const double* p, int id) {
  return __ldcg(reinterpret_cast<const double2*>(p) + id);
}
__device__ __forceinline__ void d2st(double* p, int id, double2 v) {
  reinterpret_cast<double2*>(p)[id] = v;
}

// node id at grid (i, j) of a level; `up`: as seen from the cells above the slit
__device__ __forceinline__ int mg_node(const DMesh& m, int i, int j, bool up) {
  if (j < 0 || j > m.ny) return -1;
  const int4 rw = __ldg(m.nrow + j);
  if (i < rw.x || i >= rw.y) return -1;
  if (up && j == m.notch_row && i >= m.notch_lo && i < m.notch_hi)
    return m.dup_start + (i - m.notch_lo);
  return rw.z + (i - rw.x);
}
__device__ __forceinline__ int mg_cell(const DMesh& m, int ci, int cj) {
  if (cj < 0 || cj >= m.ny) return -1;
  const int4 er = __ldg(m.erow + cj);
  return (ci >= er.x && ci < er.y) ? er.z + (ci - er.x) : -1;
}
__device__ __forceinline__ bool mg_dup_pos(const DMesh& m, int i, int j) {
  return m.notch_row >= 0 && j == m.notch_row && i >= m.notch_lo && i < m.notch_hi;
}
__device__ __forceinline__ bool mg_is_dup(const DMesh& m, int id) {
  return m.notch_row >= 0 && id >= m.dup_start;
}

// bilinear weight of parent corner K at child c's corner k (children (0,0),(1,0),(0,1),(1,1);
// corners CCW from (-,-))
__device__ __forceinline__ double mg_q(int c, int k, int K) {
  const int ox = c & 1, oy = c >> 1;
  const int cx = (k == 1 || k == 2), cy = (k >= 2);
  const double x = 0.5 * (ox + cx), y = 0.5 * (oy + cy);
  const int X = (K == 1 || K == 2), Y = (K >= 2);
  return (X ? x : 1.0 - x) * (Y ? y : 1.0 - y);
}

// ----------------------------------------------------------------------------------------
// Generic warp march (pf_march.cuh march_unit without the PCG specifics).  Op provides
//   double2 in(int id, int i, int j, bool dup, double& aux)  input value at a node (zero, aux 0
//                                                             for id < 0)
//   void cell(int eid, const double2 (&v)[4], const double (&a)[4], double2 (&f)[4])
//   void out(int id, double2 Av, double2 vin)                 once per owned node
template <class Op>
__device__ __forceinline__ void mg_march(const DMesh& m, const MarchGeom& G, int unit, Op& op,
                                         MgWarp& ws) {
  const int lane = threadIdx.x & 31;
  const int strip = unit % G.n_strips;
  const int r0 = (unit / G.n_strips) * G.rows_per_unit;
  const int r1 = min(r0 + G.rows_per_unit, m.ny + 1);
  const int col = strip * TXW - 1 + lane;
  const bool lane_own = lane >= 1 && lane <= TXW;
  const int R = m.notch_row;
  const bool dupcol = R >= 0 && col >= m.notch_lo && col < m.notch_hi;
  int nbase = -1000000, ebase = -1000000;
  auto nid = [&](int j) -> int {
    if (j < 0 || j > m.ny) return -1;
    if (j - nbase >= 32 || j < nbase) {
      __syncwarp();
      nbase = j;
      const int jj = j + lane;
      ws.nwin[lane] = jj <= m.ny ? __ldg(m.nrow + jj) : make_int4(0, 0, 0, 0);
      __syncwarp();
    }
    const int4 rw = ws.nwin[j - nbase];
    return (col >= rw.x && col < rw.y) ? rw.z + (col - rw.x) : -1;
  };
  auto cell_id = [&](int cj) -> int {
    if (cj < 0 || cj >= m.ny) return -1;
    if (cj - ebase >= 32 || cj < ebase) {
      __syncwarp();
      ebase = cj;
      const int jj = cj + lane;
      ws.ewin[lane] = jj < m.ny ? __ldg(m.erow + jj) : make_int4(0, 0, 0, 0);
      __syncwarp();
    }
    if (lane >= 31) return -1;
    const int4 er = ws.ewin[cj - ebase];
    return (col >= er.x && col < er.y) ? er.z + (col - er.x) : -1;
  };
  auto load_dup = [&]() {
    const int id = dupcol ? m.dup_start + (col - m.notch_lo) : -1;
    double a = 0.0;
    const double2 v = op.in(id, col, R, true, a);
    ws.dv[lane] = v;
    ws.da[lane] = a;
    ws.did[lane] = id;
    __syncwarp();
  };
  double a_lo = 0.0, a_hi = 0.0;
  int id_lo = nid(r0 - 1);
  double2 v_lo = op.in(id_lo, col, r0 - 1, false, a_lo);
  bool lo_slit = (r0 - 1 == R);
  if (lo_slit) load_dup();
  double2 acc_lo = make_double2(0.0, 0.0);
  for (int cj = r0 - 1; cj < r1; ++cj) {
    const int jh = cj + 1;
    const int id_hi = nid(jh);
    const double2 v_hi = op.in(id_hi, col, jh, false, a_hi);
    const bool hi_slit = (jh == R);
    const int eid = cell_id(cj);
    const bool use_dup = lo_slit && dupcol;
    const double2 b0 = use_dup ? ws.dv[lane] : v_lo;
    const double e0 = use_dup ? ws.da[lane] : a_lo;
    const double2 b1 = shfl_dn(b0), t2 = shfl_dn(v_hi);
    const double e1 = shfl_dn(e0), e2 = shfl_dn(a_hi);
    double2 f[4];
    f[0] = f[1] = f[2] = f[3] = make_double2(0.0, 0.0);
    if (eid >= 0) {
      const double2 v[4] = {b0, b1, t2, v_hi};
      const double a[4] = {e0, e1, e2, a_hi};
      op.cell(eid, v, a, f);
    }
    const double2 c1l = shfl_up(f[1]), c2l = shfl_up(f[2]);
    if (lane_own && cj >= r0) {
      if (use_dup) {
        if (id_lo >= 0) op.out(id_lo, acc_lo, v_lo);  // lower face: cells below only
        const int idd = ws.did[lane];
        if (idd >= 0) op.out(idd, d2add(c1l, f[0]), ws.dv[lane]);  // upper face
      } else if (id_lo >= 0) {
        op.out(id_lo, d2add(d2add(acc_lo, c1l), f[0]), v_lo);
      }
    }
    acc_lo = d2add(c2l, f[3]);
    if (hi_slit) {
      __syncwarp();
      load_dup();
    }
    v_lo = v_hi;
    a_lo = a_hi;
    id_lo = id_hi;
    lo_slit = hi_slit;
  }
}

// ---- fine-level (level 0) node ops for mg_march ---------------------------------------------
// The fine operator is K_uu(u, d) applied cell by cell (pf_march.cuh mom_cell_fast: branch bits
// per cell, g(d) at the Gauss points from the nodal d carried as the march's aux value).
struct FineBase {
  const Consts* C;
  const uint8_t* flags;
  const double* d;
  const double* dinv;
  __device__ void cell(int eid, const double2 (&v)[4], const double (&a)[4],
                       double2 (&f)[4]) const {
    mom_cell_fast(*C, v, a, __ldg(flags + eid), f);
  }
  __device__ double2 di(int id) const { return __ldg(reinterpret_cast<const double2*>(dinv) + id); }
};

__device__ __forceinline__ double2 mask2(double2 v, double2 di) {
  return make_double2(di.x != 0.0 ? v.x : 0.0, di.y != 0.0 ? v.y : 0.0);
}

struct FineResid : FineBase {  // x = omega D^-1 r (pre-smoothing from zero), t = r - A x
  double om;
  const double* r;
  double* t;
  __device__ double2 in(int id, int, int, bool, double& aux) const {
    aux = 0.0;
    if (id < 0) return make_double2(0.0, 0.0);
    aux = __ldg(d + id);
    const double2 dv = di(id), bv = d2ldcg(r, id);
    return make_double2(om * dv.x * bv.x, om * dv.y * bv.y);
  }
  __device__ void out(int id, double2 Av, double2) const {
    const double2 bv = d2ldcg(r, id);
    d2st(t, id, mask2(make_double2(bv.x - Av.x, bv.y - Av.y), di(id)));
  }
};

// prolongation (P e_{l+1}) at node (i, j) of level l; dup = upper-face slit node
__device__ __forceinline__ double2 mg_prolong(const DMesh& mf, const DMesh& mc,
                                              const double* ec, int i, int j, bool dup) {
  const bool up = dup || (mf.notch_row >= 0 && j > mf.notch_row);
  const int I0 = i >> 1, J0 = j >> 1;
  const bool ox = i & 1, oy = j & 1;
  double2 s = make_double2(0.0, 0.0);
#pragma unroll
  for (int bj = 0; bj < 2; ++bj) {
    if (bj == 1 && !oy) break;
#pragma unroll
    for (int bi = 0; bi < 2; ++bi) {
      if (bi == 1 && !ox) break;
      const int c = mg_node(mc, I0 + bi, J0 + bj, up);
      if (c < 0) continue;
      const double w = (ox ? 0.5 : 1.0) * (oy ? 0.5 : 1.0);
      const double2 v = d2ldcg(ec, c);
      s.x += w * v.x;
      s.y += w * v.y;
    }
  }
  return s;
}

struct FineSmooth : FineBase {  // y = omega D^-1 r + P e_1, z = y + omega D^-1 (r - A y); r.z
  double om;
  const double* r;
  double* z;
  const DMesh* mf;
  const DMesh* mc;
  const double* ec;
  double* rz;
  __device__ double2 in(int id, int i, int j, bool dup, double& aux) const {
    aux = 0.0;
    if (id < 0) return make_double2(0.0, 0.0);
    aux = __ldg(d + id);
    const double2 dv = di(id), bv = d2ldcg(r, id);
    const double2 pe = mg_prolong(*mf, *mc, ec, i, j, dup);
    return mask2(make_double2(om * dv.x * bv.x + pe.x, om * dv.y * bv.y + pe.y), dv);
  }
  __device__ void out(int id, double2 Av, double2 y) const {
    const double2 dv = di(id), bv = d2ldcg(r, id);
    const double2 ev = make_double2(y.x + om * dv.x * (bv.x - Av.x),
                                    y.y + om * dv.y * (bv.y - Av.y));
    d2st(z, id, ev);
    *rz += bv.x * ev.x + bv.y * ev.y;
  }
};

__device__ __forceinline__ double mg_hash01(unsigned k) {
  k ^= k >> 16; k *= 0x7feb352du; k ^= k >> 15; k *= 0x846ca68bu; k ^= k >> 16;
  return (double)(k & 0xffffff) * (1.0 / 16777216.0) - 0.5;
}

struct FinePow : FineBase {  // power step vout = D^-1 A vin (vin == nullptr: hashed start)
  const double* vin;
  double* vout;
  __device__ double2 in(int id, int, int, bool, double& aux) const {
    aux = 0.0;
    if (id < 0) return make_double2(0.0, 0.0);
    aux = __ldg(d + id);
    const double2 v = vin ? d2ldcg(vin, id)
                          : make_double2(mg_hash01(2u * id + 1u), mg_hash01(2u * id + 2u));
    return mask2(v, di(id));
  }
  __device__ void out(int id, double2 Av, double2) const {
    const double2 dv = di(id);
    d2st(vout, id, make_double2(dv.x * Av.x, dv.y * Av.y));
  }
};

struct FinePcg : FineBase {  // p = z + beta p_old (owner stores), q = A p (masked), p.q
  double beta;
  const double* z;
  const double* pold;
  double* pnew;
  double* q;
  double* pq;
  __device__ double2 in(int id, int, int, bool, double& aux) const {
    aux = 0.0;
    if (id < 0) return make_double2(0.0, 0.0);
    aux = __ldg(d + id);
    const double2 zv = d2ldcg(z, id);
    if (!pold) return zv;
    const double2 po = d2ldcg(pold, id);
    return make_double2(zv.x + beta * po.x, zv.y + beta * po.y);
  }
  __device__ void out(int id, double2 Av, double2 p) const {
    const double2 qv = mask2(Av, di(id));
    d2st(pnew, id, p);
    d2st(q, id, qv);
    *pq += p.x * qv.x + p.y * qv.y;
  }
};

// ---- coarse levels: node-parallel phases ----------------------------------------------------
// Visit every node of a level: items are (node row or the slit-duplicate row, 32-column chunk);
// f(id, i, j, dup) per existing node.  worker/nw count warps.
template <class F>
__device__ __forceinline__ void mg_for_nodes(const DMesh& m, int worker, int nw, F&& f) {
  const int lane = threadIdx.x & 31;
  const int chunks = (m.nx + 1 + 31) / 32;
  const int rows = m.ny + 1 + (m.notch_row >= 0 ? 1 : 0);
  for (int it = worker; it < rows * chunks; it += nw) {
    const int row = it / chunks, i = (it % chunks) * 32 + lane;
    if (row <= m.ny) {
      const int id = mg_node(m, i, row, false);
      if (id >= 0) f(id, i, row, false);
    } else if (i >= m.notch_lo && i < m.notch_hi) {
      f(m.dup_start + (i - m.notch_lo), i, m.notch_row, true);
    }
  }
}
__host__ __device__ inline int mg_items(int nx, int ny, bool notch) {
  return (ny + 1 + (notch ? 1 : 0)) * ((nx + 1 + 31) / 32);
}

// restriction (P^T t_{l-1}) at node (I, J, up) of level l >= 1: gather over the <= 9 fine
// nodes that interpolate from it (a fine node on the far side of the slit does not)
__device__ __forceinline__ double2 mg_restrict_at(const DMesh& mf, const DMesh& mc,
                                                  const double* t, int I, int J, bool up) {
  const int Rf = mf.notch_row;
  const bool dpos = mg_dup_pos(mc, I, J);
  double2 s = make_double2(0.0, 0.0);
#pragma unroll
  for (int b = -1; b <= 1; ++b) {
    const int j = 2 * J + b;
    const double wy = b ? 0.5 : 1.0;
#pragma unroll
    for (int a = -1; a <= 1; ++a) {
      const int i = 2 * I + a;
      const double w = wy * (a ? 0.5 : 1.0);
      const int fr = mg_node(mf, i, j, false);
      if (fr < 0) continue;
      const bool s_reg = Rf >= 0 && j > Rf;
      if (!dpos || s_reg == up) {
        const double2 v = d2ldcg(t, fr);
        s.x += w * v.x;
        s.y += w * v.y;
      }
      if (mg_dup_pos(mf, i, j) && (!dpos || up)) {
        const double2 v = d2ldcg(t, mf.dup_start + (i - mf.notch_lo));
        s.x += w * v.x;
        s.y += w * v.y;
      }
    }
  }
  return s;
}

// Matrix-vector product of a coarse level at one node, gathered from its <= 4 cells (stored
// Galerkin matrices).  The 3x3 neighbourhood is looked up the way each cell sees its corners
// (bottom corners from above the slit, top corners from below), so the slit faces separate:
// slots 0-2 row j-1, 3-5 row j seen from the cells below, 6-8 row j from the cells above,
// 9-11 row j+1.  xval(id) gives the input vector at a node; the cells are summed in the fixed
// order below-left, below-right, above-left, above-right.  xc = input at the node itself.
template <class X>
__device__ __forceinline__ double2 mg_gather(const DMesh& m, const double* K, int id, int i,
                                             int j, X&& xval, double2& xc) {
  int nid[12];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    nid[a] = mg_node(m, i + a - 1, j - 1, true);
    nid[3 + a] = mg_node(m, i + a - 1, j, false);
    nid[6 + a] = mg_node(m, i + a - 1, j, true);
    nid[9 + a] = mg_node(m, i + a - 1, j + 1, false);
  }
  double2 xv[12];
#pragma unroll
  for (int sl = 0; sl < 12; ++sl) {
    const int row = sl / 3;
    if (row == 2 && nid[sl] == nid[sl - 3]) {
      xv[sl] = xv[sl - 3];
      continue;
    }
    xv[sl] = nid[sl] >= 0 ? xval(nid[sl]) : make_double2(0.0, 0.0);
  }
  const bool below = nid[4] == id, above = nid[7] == id;
  xc = below ? xv[4] : xv[7];
  // cells: (dx, dy, corner of this node, corner slots 0..3)
  const int cdx[4] = {-1, 0, -1, 0}, cdy[4] = {-1, -1, 0, 0}, ck[4] = {2, 3, 1, 0};
  const int cs[4][4] = {{0, 1, 4, 3}, {1, 2, 5, 4}, {6, 7, 10, 9}, {7, 8, 11, 10}};
  double2 acc = make_double2(0.0, 0.0);
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    if (q < 2 ? !below : !above) continue;
    const int e = mg_cell(m, i + cdx[q], j + cdy[q]);
    if (e < 0) continue;
    const int k = ck[q];
    const double2* Kr = reinterpret_cast<const double2*>(K + 64 * (size_t)e);
#pragma unroll
    for (int bq = 0; bq < 4; ++bq) {
      const double2 v = xv[cs[q][bq]];
      const double2 kx = __ldcg(Kr + (2 * k) * 4 + bq), ky = __ldcg(Kr + (2 * k + 1) * 4 + bq);
      acc.x += kx.x * v.x + kx.y * v.y;
      acc.y += ky.x * v.x + ky.y * v.y;
    }
  }
  return acc;
}

// ---- setup helpers ----------------------------------------------------------------------------
// Galerkin cell matrices of level lc from level lc-1 (lc == 1: from the matrix-free fine
// operator, masked at the Dirichlet dofs); one warp per coarse cell
__device__ __forceinline__ void mg_galerkin(const MgArgs& A, int lc, int worker, int nw,
                                            MgGal& sg) {
  const DMesh& mc = A.L[lc].m;
  const DMesh& mf = A.L[lc - 1].m;
  const int lane = threadIdx.x & 31;
  const int c = lane >> 3, bcol = lane & 7;
  const int ox = c & 1, oy = c >> 1;
  double* KE = A.L[lc].K;
  for (int it = worker; it < mc.ny * mc.nx; it += nw) {  // one coarse cell per warp item
    const int J = it / mc.nx;
    const int4 er = __ldg(mc.erow + J);
    {
      const int I = it % mc.nx;
      if (I < er.x || I >= er.y) continue;  // warp-uniform
      const int E = er.z + (I - er.x);
      const int ci = 2 * I + ox, cj = 2 * J + oy;
      // column bcol of child c's (masked) cell matrix
      double col[8];
      if (lc == 1) {
        int n[4];
        n[0] = mg_node(mf, ci, cj, true);
        n[1] = mg_node(mf, ci + 1, cj, true);
        n[2] = mg_node(mf, ci + 1, cj + 1, false);
        n[3] = mg_node(mf, ci, cj + 1, false);
        const int fe = mg_cell(mf, ci, cj);
        double2 di[4];
        double dc[4];
        double2 v[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          di[q] = n[q] >= 0 ? __ldg(reinterpret_cast<const double2*>(A.L[0].dinv) + n[q])
                            : make_double2(0.0, 0.0);
          dc[q] = n[q] >= 0 ? __ldg(A.d + n[q]) : 0.0;
          v[q] = make_double2(bcol == 2 * q ? 1.0 : 0.0, bcol == 2 * q + 1 ? 1.0 : 0.0);
        }
        const double fb = (bcol & 1) ? di[bcol >> 1].y : di[bcol >> 1].x;
        double2 f[4];
        f[0] = f[1] = f[2] = f[3] = make_double2(0.0, 0.0);
        if (fe >= 0 && fb != 0.0) mom_cell_fast(A.C, v, dc, __ldg(A.flags + fe), f);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          col[2 * q] = di[q].x != 0.0 ? f[q].x : 0.0;
          col[2 * q + 1] = di[q].y != 0.0 ? f[q].y : 0.0;
        }
      } else {
        const int fe = mg_cell(mf, ci, cj);
        const double* Kf = A.L[lc - 1].K + 64 * (size_t)fe;
#pragma unroll
        for (int a = 0; a < 8; ++a) col[a] = fe >= 0 ? __ldcg(Kf + a * 8 + bcol) : 0.0;
      }
#pragma unroll
      for (int a = 0; a < 8; ++a) sg.Kc[c][a * 8 + bcol] = col[a];
      __syncwarp();
      {  // T_c = K_c Q_c: lane (c, a = bcol) computes row a
        const int a = bcol;
        double tr[8];
#pragma unroll
        for (int B = 0; B < 8; ++B) {
          double s = 0.0;
#pragma unroll
          for (int k2 = 0; k2 < 4; ++k2) s += sg.Kc[c][a * 8 + 2 * k2 + (B & 1)] * mg_q(c, k2, B >> 1);
          tr[B] = s;
        }
#pragma unroll
        for (int B = 0; B < 8; ++B) sg.T[c][a * 8 + B] = tr[B];
      }
      __syncwarp();
#pragma unroll
      for (int h = 0; h < 2; ++h) {  // K_E = sum_c Q_c^T T_c: entries lane, lane + 32
        const int e = lane + 32 * h;
        const int Ar = e >> 3, B = e & 7;
        double s = 0.0;
#pragma unroll
        for (int cc = 0; cc < 4; ++cc)
#pragma unroll
          for (int k2 = 0; k2 < 4; ++k2)
            s += mg_q(cc, k2, Ar >> 1) * sg.T[cc][(2 * k2 + (Ar & 1)) * 8 + B];
        KE[64 * (size_t)E + e] = s;
      }
      __syncwarp();
    }
  }
}

__device__ __forceinline__ void mg_diag(const MgArgs& A, int l, int worker, int nw) {
  const DMesh& m = A.L[l].m;
  const double* K = A.L[l].K;
  mg_for_nodes(m, worker, nw, [&](int id, int i, int j, bool dup) {
    double sx = 0.0, sy = 0.0;
    // (cell dx, dy, corner of this node in it)
    const int cdx[4] = {-1, 0, -1, 0}, cdy[4] = {-1, -1, 0, 0}, ck[4] = {2, 3, 1, 0};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int ci = i + cdx[q], cj = j + cdy[q];
      const int e = mg_cell(m, ci, cj);
      if (e < 0) continue;
      // the node must be this cell's corner ck[q] (slit faces)
      const int k = ck[q];
      const int ni = ci + ((k == 1 || k == 2) ? 1 : 0), nj = cj + (k >= 2 ? 1 : 0);
      const int nid = mg_node(m, ni, nj, k < 2);
      if (nid != id) continue;
      sx += __ldcg(K + 64 * (size_t)e + (2 * k) * 9);
      sy += __ldcg(K + 64 * (size_t)e + (2 * k + 1) * 9);
    }
    (void)dup;
    d2st(A.L[l].dinv, id, make_double2(sx > 0.0 ? 1.0 / sx : 0.0, sy > 0.0 ? 1.0 / sy : 0.0));
  });
}

// ---- coarse-level phases (levels >= 1; worker / nw count warps) ------------------------------
// restriction b_l = P^T t_{l-1} (masked at dead dofs)
__device__ __forceinline__ void mg_restrict(const MgArgs& A, int l, int worker, int nw) {
  const MgLevel& L = A.L[l];
  const DMesh& mf = A.L[l - 1].m;
  const double* tf = A.L[l - 1].t;
  mg_for_nodes(L.m, worker, nw, [&](int id, int i, int j, bool dup) {
    d2st(L.b, id, mask2(mg_restrict_at(mf, L.m, tf, i, j, dup), d2ldcg(L.dinv, id)));
  });
}
// down-sweep residual t = b - A x with x = omega D^-1 b (one Jacobi sweep from zero)
__device__ __forceinline__ void mg_resid(const MgArgs& A, int l, double om, int worker, int nw) {
  const MgLevel& L = A.L[l];
  mg_for_nodes(L.m, worker, nw, [&](int id, int i, int j, bool) {
    auto xval = [&](int n) -> double2 {
      const double2 di = d2ldcg(L.dinv, n), bv = d2ldcg(L.b, n);
      return make_double2(om * di.x * bv.x, om * di.y * bv.y);
    };
    double2 xc;
    const double2 Av = mg_gather(L.m, L.K, id, i, j, xval, xc);
    const double2 di = d2ldcg(L.dinv, id), bv = d2ldcg(L.b, id);
    d2st(L.t, id, mask2(make_double2(bv.x - Av.x, bv.y - Av.y), di));
  });
}
// prolongation y = omega D^-1 b + P e_{l+1} (into t)
__device__ __forceinline__ void mg_prolongate(const MgArgs& A, int l, double om, int worker,
                                              int nw) {
  const MgLevel& L = A.L[l];
  const MgLevel& Lc = A.L[l + 1];
  mg_for_nodes(L.m, worker, nw, [&](int id, int i, int j, bool dup) {
    const double2 di = d2ldcg(L.dinv, id), bv = d2ldcg(L.b, id);
    const double2 pe = mg_prolong(L.m, Lc.m, Lc.e, i, j, dup);
    d2st(L.t, id, mask2(make_double2(om * di.x * bv.x + pe.x, om * di.y * bv.y + pe.y), di));
  });
}
// post-smoothing e = y + omega D^-1 (b - A y), y in t
__device__ __forceinline__ void mg_smooth(const MgArgs& A, int l, double om, int worker, int nw) {
  const MgLevel& L = A.L[l];
  mg_for_nodes(L.m, worker, nw, [&](int id, int i, int j, bool) {
    auto xval = [&](int n) -> double2 { return d2ldcg(L.t, n); };
    double2 y;
    const double2 Av = mg_gather(L.m, L.K, id, i, j, xval, y);
    const double2 di = d2ldcg(L.dinv, id), bv = d2ldcg(L.b, id);
    d2st(L.e, id, make_double2(y.x + om * di.x * (bv.x - Av.x), y.y + om * di.y * (bv.y - Av.y)));
  });
}
// Jacobi sweep eout = ein + omega D^-1 (b - A ein)
__device__ __forceinline__ void mg_sweep(const MgArgs& A, int l, double om, const double* ein,
                                         double* eout, int worker, int nw) {
  const MgLevel& L = A.L[l];
  mg_for_nodes(L.m, worker, nw, [&](int id, int i, int j, bool) {
    auto xval = [&](int n) -> double2 { return d2ldcg(ein, n); };
    double2 x;
    const double2 Av = mg_gather(L.m, L.K, id, i, j, xval, x);
    const double2 di = d2ldcg(L.dinv, id), bv = d2ldcg(L.b, id);
    d2st(eout, id, make_double2(x.x + om * di.x * (bv.x - Av.x), x.y + om * di.y * (bv.y - Av.y)));
  });
}
// power step vout = D^-1 A vin (vin == nullptr: hashed start vector)
__device__ __forceinline__ void mg_pow(const MgArgs& A, int l, const double* vin, double* vout,
                                       int worker, int nw) {
  const MgLevel& L = A.L[l];
  mg_for_nodes(L.m, worker, nw, [&](int id, int i, int j, bool) {
    auto xval = [&](int n) -> double2 {
      const double2 di = d2ldcg(L.dinv, n);
      const double2 v = vin ? d2ldcg(vin, n)
                            : make_double2(mg_hash01(2u * n + 1u), mg_hash01(2u * n + 2u));
      return mask2(v, di);
    };
    double2 x;
    const double2 Av = mg_gather(L.m, L.K, id, i, j, xval, x);
    const double2 di = d2ldcg(L.dinv, id);
    d2st(vout, id, make_double2(di.x * Av.x, di.y * Av.y));
  });
}

// coarsest level: b = P^T t, then the dense inverse or nu_c Jacobi sweeps from zero (a
// symmetric polynomial in D^-1 A times D^-1, so the V-cycle stays symmetric); result in L.e.
// Runs inside one CTA (the tail kernel).
__device__ __forceinline__ void mg_coarse_cta(const MgArgs& A, double om) {
  const int c = A.n_levels - 1;
  const MgLevel& L = A.L[c];
  const int nd = 2 * L.m.n_nodes;
  const int w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  mg_restrict(A, c, w, nw);
  __syncthreads();
  if (A.dense) {
    for (int i = threadIdx.x; i < nd; i += blockDim.x) {
      double s = 0.0;
      for (int j = 0; j < nd; ++j) s += __ldcg(A.Ainv + (size_t)i * nd + j) * __ldcg(L.b + j);
      L.e[i] = s;
    }
    __syncthreads();
    return;
  }
  double* bufs[2] = {L.e, L.t};
  int cur = (A.nu_c - 1) % 2 == 0 ? 0 : 1;  // the last sweep lands in L.e
  for (int i = threadIdx.x; i < nd; i += blockDim.x)
    bufs[cur][i] = om * __ldcg(L.dinv + i) * __ldcg(L.b + i);
  __syncthreads();
  for (int s = 1; s < A.nu_c; ++s) {
    mg_sweep(A, c, om, bufs[cur], bufs[cur ^ 1], w, nw);
    cur ^= 1;
    __syncthreads();
  }
}

// ---- deterministic grid reductions: per-CTA partials, the last CTA sums them in order --------
template <int NV>
__device__ __forceinline__ void mg_block_sum(double (&v)[NV], double* red) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < NV; ++k) v[k] = warp_sum(v[k]);
  if (lane == 0)
#pragma unroll
    for (int k = 0; k < NV; ++k) red[wid * NV + k] = v[k];
  __syncthreads();
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      double s = 0.0;
      for (int q = 0; q < (int)(blockDim.x >> 5); ++q) s += red[q * NV + k];
      v[k] = s;
    }
  }
  __syncthreads();
}
// every CTA reduces all partials (fixed order) -> identical totals in every CTA
template <int NV>
__device__ __forceinline__ void mg_all_reduce(const double* part, int nparts, double* red,
                                              double (&out)[NV]) {
  if (threadIdx.x < 32) {
    double s[NV];
#pragma unroll
    for (int k = 0; k < NV; ++k) s[k] = 0.0;
    for (int i = threadIdx.x; i < nparts; i += 32)
#pragma unroll
      for (int k = 0; k < NV; ++k) s[k] += __ldcg(part + NV * i + k);
#pragma unroll
    for (int k = 0; k < NV; ++k) s[k] = warp_sum(s[k]);
    if (threadIdx.x == 0)
#pragma unroll
      for (int k = 0; k < NV; ++k) red[k] = s[k];
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < NV; ++k) out[k] = red[k];
  __syncthreads();
}
// writes this CTA's partials; returns true in the last CTA to arrive (after a fence)
template <int NV>
__device__ __forceinline__ bool mg_publish(double (&v)[NV], double* part, unsigned int* count,
                                           double* red) {
  mg_block_sum<NV>(v, red);
  __shared__ bool last;
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < NV; ++k) part[NV * blockIdx.x + k] = v[k];
    __threadfence();
    last = atomicAdd(count, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (last) __threadfence();
  return last;
}

// ================================================================================================
// kernels of one solve: k_mg_init, WHILE { fine resid, (restrict, resid) per grid level, tail,
// (prolongate, smooth) per grid level, fine smooth, pcg, update }, k_mg_finish
__global__ void __launch_bounds__(MG_NT) k_mg_init(MgArgs A) {
  __shared__ double red[MG_WARPS];
  double rr = 0.0;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < A.ndof;
       i += (long long)gridDim.x * blockDim.x) {
    const double v = __ldcg(A.r + i);
    rr += v * v;
    A.x[i] = 0.0;
  }
  double v[1] = {rr};
  if (mg_publish<1>(v, A.part, &A.ctl->count, red)) {
    double tot[1];
    mg_all_reduce<1>(A.part, gridDim.x, red, tot);
    if (threadIdx.x == 0) {
      MgCtl& c = *A.ctl;
      c.count = 0;
      c.rr = tot[0];
      const volatile MgIn* in = A.in;
      c.maxiter = in->maxiter;
      c.target = in->target;
      c.bnorm = sqrt(tot[0]);
      c.atol = in->rtol * c.bnorm;
      c.k = 0;
      c.rho_prev = 0.0;
      c.status = CG_CONVERGED;
      // scipy cg: b == 0 returns x = 0; otherwise the loop tests ||r|| < atol first
      c.done = (c.bnorm == 0.0 || sqrt(tot[0]) < c.atol) ? 1 : 0;
      if (!c.done && c.maxiter <= 0) { c.done = 1; c.status = CG_MAXITER; }
      if (A.use_cond) cudaGraphSetConditional(A.cond, c.done ? 0u : 1u);
    }
  }
}

__global__ void __launch_bounds__(MG_NT, 2) k_mg_fine_resid(MgArgs A) {
  __shared__ MgWarp ws[MG_WARPS];
  const double om = __ldcg(&A.ctl->omega[0]);
  FineResid op{{&A.C, A.flags, A.d, A.L[0].dinv}, om, A.r, A.L[0].t};
  const int w = blockIdx.x * MG_WARPS + (threadIdx.x >> 5);
  if (w < A.g0.n_units) mg_march(A.L[0].m, A.g0, w, op, ws[threadIdx.x >> 5]);
}

__global__ void __launch_bounds__(MG_NT) k_mg_restrict(MgArgs A, int l) {
  mg_restrict(A, l, blockIdx.x * MG_WARPS + (threadIdx.x >> 5), gridDim.x * MG_WARPS);
}
__global__ void __launch_bounds__(MG_NT) k_mg_resid(MgArgs A, int l) {
  mg_resid(A, l, __ldcg(&A.ctl->omega[l]), blockIdx.x * MG_WARPS + (threadIdx.x >> 5),
           gridDim.x * MG_WARPS);
}
__global__ void __launch_bounds__(MG_NT) k_mg_prolongate(MgArgs A, int l) {
  mg_prolongate(A, l, __ldcg(&A.ctl->omega[l]), blockIdx.x * MG_WARPS + (threadIdx.x >> 5),
                gridDim.x * MG_WARPS);
}
__global__ void __launch_bounds__(MG_NT) k_mg_smooth(MgArgs A, int l) {
  mg_smooth(A, l, __ldcg(&A.ctl->omega[l]), blockIdx.x * MG_WARPS + (threadIdx.x >> 5),
            gridDim.x * MG_WARPS);
}

// levels [n_tail, n_levels) in one CTA: the V-cycle below level n_tail - 1 (result e_{n_tail})
__global__ void __launch_bounds__(MG_TAIL_NT) k_mg_tail(MgArgs A) {
  const int w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int nl = A.n_levels, l0 = A.n_tail;
  for (int l = l0; l < nl - 1; ++l) {
    mg_restrict(A, l, w, nw);
    __syncthreads();
    mg_resid(A, l, __ldcg(&A.ctl->omega[l]), w, nw);
    __syncthreads();
  }
  mg_coarse_cta(A, __ldcg(&A.ctl->omega[nl - 1]));
  for (int l = nl - 2; l >= l0; --l) {
    const double om = __ldcg(&A.ctl->omega[l]);
    mg_prolongate(A, l, om, w, nw);
    __syncthreads();
    mg_smooth(A, l, om, w, nw);
    __syncthreads();
  }
}

__global__ void __launch_bounds__(MG_NT, 2) k_mg_fine_smooth(MgArgs A) {
  __shared__ MgWarp ws[MG_WARPS];
  __shared__ double red[MG_WARPS];
  const double om = __ldcg(&A.ctl->omega[0]);
  double rz = 0.0;
  FineSmooth op{{&A.C, A.flags, A.d, A.L[0].dinv}, om, A.r, A.z, &A.L[0].m, &A.L[1].m,
                A.L[1].e, &rz};
  const int w = blockIdx.x * MG_WARPS + (threadIdx.x >> 5);
  if (w < A.g0.n_units) mg_march(A.L[0].m, A.g0, w, op, ws[threadIdx.x >> 5]);
  double v[1] = {rz};
  mg_block_sum<1>(v, red);
  if (threadIdx.x == 0) A.part[blockIdx.x] = v[0];  // r.z partials, reduced by k_mg_pcg
}

__global__ void __launch_bounds__(MG_NT, 2) k_mg_pcg(MgArgs A, int n_rz) {
  __shared__ MgWarp ws[MG_WARPS];
  __shared__ double red[MG_WARPS];
  double rho[1];
  mg_all_reduce<1>(A.part, n_rz, red, rho);
  const long long k = __ldcg(&A.ctl->k);
  const bool first = k == 0;
  double pq = 0.0;
  FinePcg op{{&A.C, A.flags, A.d, A.L[0].dinv}, first ? 0.0 : rho[0] / __ldcg(&A.ctl->rho_prev),
             A.z, first ? nullptr : ((k & 1) ? A.p0 : A.p1), (k & 1) ? A.p1 : A.p0, A.q, &pq};
  const int w = blockIdx.x * MG_WARPS + (threadIdx.x >> 5);
  if (w < A.g0.n_units) mg_march(A.L[0].m, A.g0, w, op, ws[threadIdx.x >> 5]);
  double v[1] = {pq};
  mg_block_sum<1>(v, red);
  if (threadIdx.x == 0) A.part[n_rz + blockIdx.x] = v[0];  // p.q partials after the r.z ones
}

__global__ void __launch_bounds__(MG_NT) k_mg_update(MgArgs A, int n_rz, int n_pq) {
  __shared__ double red[MG_WARPS];
  double rho[1], pq[1];
  mg_all_reduce<1>(A.part, n_rz, red, rho);
  mg_all_reduce<1>(A.part + n_rz, n_pq, red, pq);
  const long long k = __ldcg(&A.ctl->k);
  const double alpha = rho[0] / pq[0];
  const double2* p2 = reinterpret_cast<const double2*>((k & 1) ? A.p1 : A.p0);
  const double2* q2 = reinterpret_cast<const double2*>(A.q);
  double2* x2 = reinterpret_cast<double2*>(A.x);
  double2* r2 = reinterpret_cast<double2*>(A.r);
  double rr = 0.0;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < (A.ndof >> 1);
       i += (long long)gridDim.x * blockDim.x) {
    const double2 pv = __ldcg(p2 + i), qv = __ldcg(q2 + i);
    double2 xv = __ldcg(x2 + i), rv = __ldcg(r2 + i);
    xv.x += alpha * pv.x; xv.y += alpha * pv.y;
    rv.x -= alpha * qv.x; rv.y -= alpha * qv.y;
    x2[i] = xv;
    r2[i] = rv;
    rr += rv.x * rv.x + rv.y * rv.y;
  }
  double* part = A.part + n_rz + n_pq;
  double v[1] = {rr};
  if (mg_publish<1>(v, part, &A.ctl->count, red)) {
    double tot[1];
    mg_all_reduce<1>(part, gridDim.x, red, tot);
    if (threadIdx.x == 0) {
      MgCtl& c = *A.ctl;
      c.count = 0;
      c.rr = tot[0];
      c.rho_prev = rho[0];
      c.k = k + 1;
      const double rn = sqrt(tot[0]);
      if (rn < c.atol) { c.done = 1; c.status = CG_CONVERGED; }
      else if (!(rn == rn)) { c.done = 1; c.status = CG_NAN; }
      else if (c.k >= c.maxiter) { c.done = 1; c.status = CG_MAXITER; }
      if (A.use_cond) cudaGraphSetConditional(A.cond, c.done ? 0u : 1u);
    }
  }
}

__global__ void __launch_bounds__(MG_NT) k_mg_finish(MgArgs A) {
  const MgCtl& c = *A.ctl;
  const int status = __ldcg(&c.status);
  double* target = *(double* volatile*)&c.target;
  if (target && status == CG_CONVERGED)
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < A.ndof;
         i += (long long)gridDim.x * blockDim.x)
      target[i] += __ldcg(A.x + i);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    A.result->iters = __ldcg(&c.k);
    A.result->status = status;
    A.result->bnorm = __ldcg(&c.bnorm);
    A.result->rnorm = sqrt(__ldcg(&c.rr));
  }
}

// ================================================================================================
// setup kernels: Galerkin cell matrices, inverse diagonals, lambda_max by power steps, dense
// inverse of the coarsest level
__global__ void __launch_bounds__(MG_NT) k_mg_galerkin(MgArgs A, int lc) {
  __shared__ MgGal sg[MG_WARPS];
  mg_galerkin(A, lc, blockIdx.x * MG_WARPS + (threadIdx.x >> 5), gridDim.x * MG_WARPS,
              sg[threadIdx.x >> 5]);
}
__global__ void __launch_bounds__(MG_NT) k_mg_diag(MgArgs A, int l) {
  mg_diag(A, l, blockIdx.x * MG_WARPS + (threadIdx.x >> 5), gridDim.x * MG_WARPS);
}
// power step k (1..MG_POW): blocks [0, fine_blocks) march the fine level, the rest gather the
// coarse levels (concatenated item space)
__global__ void __launch_bounds__(MG_NT, 2) k_mg_pow(MgArgs A, int step, int fine_blocks) {
  __shared__ MgWarp ws[MG_WARPS];
  const int warp = threadIdx.x >> 5;
  auto vin = [&](const MgLevel& L) -> const double* {
    return step == 1 ? nullptr : (((step - 1) & 1) ? L.t : L.e);
  };
  auto vout = [&](const MgLevel& L) -> double* { return (step & 1) ? L.t : L.e; };
  if ((int)blockIdx.x < fine_blocks) {
    FinePow op{{&A.C, A.flags, A.d, A.L[0].dinv}, vin(A.L[0]), vout(A.L[0])};
    const int w = blockIdx.x * MG_WARPS + warp;
    if (w < A.g0.n_units) mg_march(A.L[0].m, A.g0, w, op, ws[warp]);
    return;
  }
  const int w = (blockIdx.x - fine_blocks) * MG_WARPS + warp;
  if (w >= A.coarse_items) return;
  int l = 1;
  while (l + 1 < A.n_levels && w >= A.L[l + 1].item_off) ++l;
  const MgLevel& L = A.L[l];
  mg_pow(A, l, vin(L), vout(L), w - L.item_off, L.items);
}
// omega_l = 4 / (3 lambda_l), lambda_l = ||v_POW|| / ||v_POW-1|| (per-level partials)
__global__ void __launch_bounds__(MG_NT) k_mg_lambda(MgArgs A) {
  __shared__ double red[MG_WARPS * 2 * MG_MAXL];
  double v[2 * MG_MAXL];
#pragma unroll
  for (int l = 0; l < 2 * MG_MAXL; ++l) v[l] = 0.0;
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long nth = (long long)gridDim.x * blockDim.x;
#pragma unroll
  for (int l = 0; l < MG_MAXL; ++l) {
    if (l >= A.n_levels) break;
    const double* a1 = (MG_POW & 1) ? A.L[l].t : A.L[l].e;
    const double* a0 = (MG_POW & 1) ? A.L[l].e : A.L[l].t;
    const long long n = 2LL * A.L[l].m.n_nodes;
    for (long long i = tid; i < n; i += nth) {
      const double x1 = __ldcg(a1 + i), x0 = __ldcg(a0 + i);
      v[2 * l] += x1 * x1;
      v[2 * l + 1] += x0 * x0;
    }
  }
  if (mg_publish<2 * MG_MAXL>(v, A.part, &A.ctl->count, red)) {
    double g[2 * MG_MAXL];
    mg_all_reduce<2 * MG_MAXL>(A.part, gridDim.x, red, g);
    if (threadIdx.x < MG_MAXL) {
      const int l = threadIdx.x;
      const double lam = (l < A.n_levels && g[2 * l + 1] > 0.0) ? sqrt(g[2 * l] / g[2 * l + 1]) : 1.0;
      A.ctl->omega[l] = 4.0 / (3.0 * (lam > 0.0 ? lam : 1.0));
    }
    if (threadIdx.x == 0) A.ctl->count = 0;
  }
}
// dense inverse of the coarsest level (one CTA): assemble from its cell matrices, Gauss-Jordan
// without pivoting (SPD on the live dofs; dead dofs get identity rows, zeroed afterwards)
__global__ void __launch_bounds__(MG_NT) k_mg_dense(MgArgs A) {
  __shared__ double M[MG_DENSE_MAX * MG_DENSE_MAX];
  __shared__ double F[MG_DENSE_MAX];
  __shared__ int live[MG_DENSE_MAX];
  const int c = A.n_levels - 1;
  const DMesh& m = A.L[c].m;
  const int nd = 2 * m.n_nodes;
  for (int ij = threadIdx.x; ij < nd * nd; ij += blockDim.x) {
    const int i = ij / nd, j = ij % nd;
    const int ni = i >> 1, nj = j >> 1, ci = i & 1, cj = j & 1;
    double s = 0.0;
    for (int cjr = 0; cjr < m.ny; ++cjr) {
      const int4 er = __ldg(m.erow + cjr);
      for (int cir = er.x; cir < er.y; ++cir) {
        const int e = er.z + (cir - er.x);
        int n[4];
        n[0] = mg_node(m, cir, cjr, true);
        n[1] = mg_node(m, cir + 1, cjr, true);
        n[2] = mg_node(m, cir + 1, cjr + 1, false);
        n[3] = mg_node(m, cir, cjr + 1, false);
        int ka = -1, kb = -1;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          if (n[q] == ni) ka = q;
          if (n[q] == nj) kb = q;
        }
        if (ka >= 0 && kb >= 0)
          s += __ldcg(A.L[c].K + 64 * (size_t)e + (2 * ka + ci) * 8 + 2 * kb + cj);
      }
    }
    M[ij] = s;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < nd; i += blockDim.x) live[i] = M[i * nd + i] > 0.0;
  __syncthreads();
  for (int ij = threadIdx.x; ij < nd * nd; ij += blockDim.x) {
    const int i = ij / nd, j = ij % nd;
    if (!live[i] || !live[j]) M[ij] = (i == j) ? 1.0 : 0.0;
  }
  __syncthreads();
  for (int k = 0; k < nd; ++k) {
    for (int i = threadIdx.x; i < nd; i += blockDim.x) F[i] = M[i * nd + k];
    __syncthreads();
    const double piv = F[k];
    for (int j = threadIdx.x; j < nd; j += blockDim.x)
      M[k * nd + j] = (j == k ? 1.0 : M[k * nd + j]) / piv;
    __syncthreads();
    for (int ij = threadIdx.x; ij < nd * nd; ij += blockDim.x) {
      const int i = ij / nd, j = ij % nd;
      if (i != k) M[ij] = (j == k ? 0.0 : M[ij]) - F[i] * M[k * nd + j];
    }
    __syncthreads();
  }
  for (int ij = threadIdx.x; ij < nd * nd; ij += blockDim.x) {
    const int i = ij / nd, j = ij % nd;
    A.Ainv[ij] = (live[i] && live[j]) ? M[ij] : 0.0;
  }
}

}  // namespace pfb
