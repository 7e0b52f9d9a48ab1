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
#include <type_traits>

// FineSmooth with its out() data prefetched (124 registers already: off unless it fits)
#ifndef PFB_SMOOTH_OPRE
#define PFB_SMOOTH_OPRE 1
#endif

namespace pfb {

constexpr int MG_MAXL = 14;
constexpr int MG_NT = 256;
constexpr int MG_WARPS = MG_NT / 32;
constexpr int MG_POW = 8;          // power steps for lambda_max(D^-1 A_l)
constexpr int MG_DENSE_MAX = 64;   // coarsest level by a dense inverse when 2 n_nodes <= this
constexpr int MG_TAIL_NT = 1024;   // threads of the single-CTA tail kernel
constexpr int MG_NS = 10;          // assembled stencil slots per node (3x3 + slit-tip face)
constexpr int MG_TAIL_P = 2;       // node passes of the tail's top level (MG_TAIL_NT / 4 each)

struct MgLevel {
  DMesh m;        // row tables (nrow/erow), notch, n_nodes/n_elems of this level
  double* K;      // [n_elems][64] Galerkin cell matrices (l >= 1)
  double* dinv;   // [2 n_nodes] inverse diagonal (0 = constrained / dead dof)
  double* b;      // right-hand side (l >= 1)
  double* t;      // residual / prolongated iterate / power-iteration buffer
  double* e;      // correction / power-iteration buffer
  int items;      // node items (rows x 32-column chunks) of mg_for_nodes
  int item_off;   // first thread of this level in the power steps' coarse thread space
  int lpn;        // lanes per node of the level's node kernels (1 | 4 | 16)
  int scalar;     // phase field (phys 1): only the xx entry of each 2x2 block is non-zero
  int s32;        // grid-level stencil products from the FP32 copy Sf (default) or from S
  // assembled form (l >= 1), slot-major: nbr [MG_NS][n] neighbour ids, S [MG_NS*4][n] 2x2
  // blocks (xx, xy, yx, yy); rid [12][n] restriction sources on level l-1; pid [4][n]
  // prolongation sources on level l+1 (l <= n_levels-2)
  const int* nbr;
  double* S;
  float* Sf;      // S rounded to FP32 for the grid-level kernels, [MG_NS][n] float4 blocks (s32;
                  // the tail keeps S)
  const int* rid;
  const int* pid;
};

// device-side control block of one solve
constexpr int MG_WARM = 3;  // warm-start directions (backward-difference table, pf_cg.cuh)
struct MgIn {  // per-solve inputs (device copy of a pinned host struct, refreshed per solve)
  double rtol;
  long long maxiter;
  double* target;                 // optional: target += x at the end
  const double* guess[MG_WARM];   // warm start: x0 = sum y_k guess[k], Galerkin-optimal y
  int n_guess;
  int probe;                      // SPD probe (pf_mgs.cuh): stop with CG_INDEFINITE at p.Ap <= 0
};
struct MgCtl {
  double omega[MG_MAXL];
  double* target;
  double rho_prev, bnorm, atol, rr;
  long long k, maxiter;
  int status, done;
  unsigned int count;  // last-block counter (reset by the last block)
};

struct MgTailSlot {  // byte offsets of one tail level in k_mg_tail's shared memory
  int nbr, rid, pid, S, dinv, b, t, e;
};

struct MgArgs {
  Consts C;
  int n_levels, n_tail;  // levels [1, n_tail) by grid kernels, [n_tail, n_levels) by k_mg_tail
  int dense, nu_c;
  MgLevel L[MG_MAXL];
  MarchGeom g0;          // march units of the fine level
  int coarse_items;      // sum of items over levels >= 1
  int phys;              // 0: momentum K_uu(u, d); 1: phase field (x component, y dead)
  const double* d;       // nodal d (level-0 momentum operator)
  const uint8_t* flags;  // level-0 tangent branch bits (momentum)
  const double* bq;      // level-0 Newton coefficient b per Gauss point [n_elems][4] (phase field)
  double *x, *r, *z, *p0, *p1, *q;
  double* Ainv;          // [nd*nd] dense inverse of the coarsest level
  double* part;          // per-CTA partial sums (>= max grid * 2 * MG_MAXL)
  MgCtl* ctl;
  const MgIn* in;
  CgResult* result;
  long long ndof;
  cudaGraphConditionalHandle cond;
  int use_cond;          // 0: launched outside the graph (unrolled profiling graph)
  long long* tclk;       // debug (PFB200_MG_TAILCLK): clock64 after each k_mg_tail phase
  MgTailSlot ts[MG_MAXL];
  int ts_ainv, ts_bytes;  // dense inverse offset, total shared memory of k_mg_tail
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
__device__ __forceinline__ double2 d2ldcg(const double* p, int id) {  // input of this kernel
  return __ldg(reinterpret_cast<const double2*>(p) + id);
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
//   struct Raw; void fetch(int id, int i, int j, bool dup, Raw&)  the node's loads (id >= 0)
//   double2 finish(const Raw&, int id, int i, int j, bool dup, double& aux)  its input value
//   double2 in(int id, int i, int j, bool dup, double& aux)  fetch + finish (zero, aux 0 for
//                                                             id < 0)
//   struct CRaw; void cfetch(int eid, CRaw&)                 the cell's own data (eid >= 0)
//   void cellr(int eid, const CRaw&, const double2 (&v)[4], const double (&a)[4],
//              double2 (&f)[4])                               the cell's contributions
//   void out(int id, double2 Av, double2 vin)                 once per owned node
//   static constexpr bool VY, AUX                             the cells read the value pair's y
//                                                             lane / the aux value of a node
// The cell data of the next cell row (branch bits / Newton coefficients) is fetched one row
// step ahead like the node rows, so no dependent HBM load sits on a row step's critical path.
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ int4 lds_int4(unsigned addr) {
  int4 v;
  asm volatile("ld.shared.v4.s32 {%0, %1, %2, %3}, [%4];\n"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr) : "memory");
  return v;
}
// optional part of an Op (overload rank by the last argument):
//   void outa(int id, double2 Av, double2 vin, double aux)   out() with the node's aux value
template <class Op>
__device__ __forceinline__ auto mg_out(Op& op, int id, double2 Av, double2 v, double a, int)
    -> decltype(op.outa(id, Av, v, a), void()) {
  op.outa(id, Av, v, a);
}
template <class Op>
__device__ __forceinline__ void mg_out(Op& op, int id, double2 Av, double2 v, double, long) {
  op.out(id, Av, v);
}
// Ops whose out() needs per-node data again (r, D^-1 of the momentum marches: both lanes of the
// value pair are taken) declare ORaw / ofetch / outp: the loads are then issued at the top of
// the row step, ahead of the cell arithmetic, instead of sitting between it and the store.
template <class Op, class = void>
struct MgOutPre {
  struct Raw {};
  __device__ static void fetch(Op&, int, Raw&) {}
  __device__ static void out(Op& op, int id, double2 Av, double2 v, double a, const Raw&) {
    mg_out(op, id, Av, v, a, 0);
  }
};
template <class Op>
struct MgOutPre<Op, std::void_t<typename Op::ORaw>> {
  using Raw = typename Op::ORaw;
  __device__ static void fetch(Op& op, int id, Raw& r) { op.ofetch(id, r); }
  __device__ static void out(Op& op, int id, double2 Av, double2 v, double, const Raw& r) {
    op.outp(id, Av, v, r);
  }
};

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
  // the row windows are read twice per row step: from 32-bit shared addresses kept in a
  // register (the generic form recomputes the warp's window address every time)
  const unsigned nwin_a = smem_u32(ws.nwin), ewin_a = smem_u32(ws.ewin);
  auto nid = [&](int j) -> int {
    if (j < 0 || j > m.ny) return -1;
    if (j - nbase >= 32 || j < nbase) {
      __syncwarp();
      nbase = j;
      const int jj = j + lane;
      ws.nwin[lane] = jj <= m.ny ? __ldg(m.nrow + jj) : make_int4(0, 0, 0, 0);
      __syncwarp();
    }
    const int4 rw = lds_int4(nwin_a + 16u * (unsigned)(j - nbase));
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
    const int4 er = lds_int4(ewin_a + 16u * (unsigned)(cj - ebase));
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
  // the next node row's loads are issued one row step ahead (Op::fetch), so every warp keeps
  // a row of loads in flight while it does the current row's FP64 work (Op::finish)
  typename Op::Raw w_hi;
  int id_hi = nid(r0);
  if (id_hi >= 0) op.fetch(id_hi, col, r0, false, w_hi);
  typename Op::CRaw c_cur;
  int e_cur = cell_id(r0 - 1);
  if (e_cur >= 0) op.cfetch(e_cur, c_cur);
  double2 acc_lo = make_double2(0.0, 0.0);
  for (int cj = r0 - 1; cj < r1; ++cj) {
    const int jh = cj + 1;
    typename MgOutPre<Op>::Raw o_lo;
    if (lane_own && cj >= r0 && id_lo >= 0) MgOutPre<Op>::fetch(op, id_lo, o_lo);
    a_hi = 0.0;
    const double2 v_hi = id_hi >= 0 ? op.finish(w_hi, id_hi, col, jh, false, a_hi)
                                    : make_double2(0.0, 0.0);
    typename Op::Raw w_nx;
    const int id_nx = (jh + 1 <= r1) ? nid(jh + 1) : -1;
    if (id_nx >= 0) op.fetch(id_nx, col, jh + 1, false, w_nx);
    const bool hi_slit = (jh == R);
    const int eid = e_cur;
    typename Op::CRaw c_nx;
    const int e_nx = (cj + 1 < r1) ? cell_id(cj + 1) : -1;
    if (e_nx >= 0) op.cfetch(e_nx, c_nx);
    const bool use_dup = lo_slit && dupcol;
    const double2 b0 = use_dup ? ws.dv[lane] : v_lo;
    const double e0 = use_dup ? ws.da[lane] : a_lo;
    // only the lanes of the value pair / the aux value that the Op's cells read travel between
    // lanes (every warp shuffle costs a convergence check as well, dead or not)
    const double2 b1 = Op::VY ? shfl_dn(b0) : make_double2(shfl_dn(b0.x), 0.0);
    const double2 t2 = Op::VY ? shfl_dn(v_hi) : make_double2(shfl_dn(v_hi.x), 0.0);
    const double e1 = Op::AUX ? shfl_dn(e0) : 0.0, e2 = Op::AUX ? shfl_dn(a_hi) : 0.0;
    double2 f[4];
    f[0] = f[1] = f[2] = f[3] = make_double2(0.0, 0.0);
    if (eid >= 0) {
      const double2 v[4] = {b0, b1, t2, v_hi};
      const double a[4] = {e0, e1, e2, a_hi};
      op.cellr(eid, c_cur, v, a, f);
    }
    const double2 c1l = Op::VY ? shfl_up(f[1]) : make_double2(shfl_up(f[1].x), 0.0);
    const double2 c2l = Op::VY ? shfl_up(f[2]) : make_double2(shfl_up(f[2].x), 0.0);
    if (lane_own && cj >= r0) {
      if (use_dup) {
        if (id_lo >= 0) MgOutPre<Op>::out(op, id_lo, acc_lo, v_lo, a_lo, o_lo);  // lower face: cells below only
        const int idd = ws.did[lane];
        if (idd >= 0) mg_out(op, idd, d2add(c1l, f[0]), ws.dv[lane], ws.da[lane], 0);  // upper face
      } else if (id_lo >= 0) {
        MgOutPre<Op>::out(op, id_lo, d2add(d2add(acc_lo, c1l), f[0]), v_lo, a_lo, o_lo);
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
    id_hi = id_nx;
    w_hi = w_nx;
    e_cur = e_nx;
    c_cur = c_nx;
  }
}

// TMA bulk copies global -> shared completing on one mbarrier (sizes and addresses are
// multiples of 16 B: the host pads every multigrid array)
__device__ __forceinline__ void mg_bulk_g2s(const void* dst, const void* src, unsigned bytes,
                                            unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
      ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mg_mbar_init_expect(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(bar)) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n"
               ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mg_mbar_wait(unsigned long long* bar, unsigned phase) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)), "r"(phase) : "memory");
}
__device__ __forceinline__ unsigned mg_r16(size_t b) { return (unsigned)((b + 15) & ~size_t(15)); }

// ---- fine-level (level 0) node ops for mg_march ---------------------------------------------
// The fine operator is K_uu(u, d) applied cell by cell (pf_march.cuh mom_cell_fast: branch bits
// per cell, g(d) at the Gauss points from the nodal d carried as the march's aux value).
struct FineBase {
  const Consts* C;
  const uint8_t* flags;
  const double* d;
  const double* dinv;
  int phys;
  const double* bq;
  struct CRaw {
    double2 b01, b23;
    unsigned fl;
  };
  __device__ void cfetch(int eid, CRaw& c) const {
    if (phys == 0) {
      c.fl = __ldg(flags + eid);
    } else {
      c.b01 = __ldg(reinterpret_cast<const double2*>(bq) + 2 * eid);
      c.b23 = __ldg(reinterpret_cast<const double2*>(bq) + 2 * eid + 1);
    }
  }
  __device__ void cell(int eid, const double2 (&v)[4], const double (&a)[4],
                       double2 (&f)[4]) const {
    CRaw c;
    cfetch(eid, c);
    cellr(eid, c, v, a, f);
  }
  __device__ void cellr(int, const CRaw& c, const double2 (&v)[4], const double (&a)[4],
                        double2 (&f)[4]) const {
    if (phys == 0) {
      mom_cell_fast(*C, v, a, c.fl, f);
    } else {  // phase field (pf_cg.cuh evo_cell_apply) on the x components
      const double2 b01 = c.b01, b23 = c.b23;
      const double pc[4] = {v[0].x, v[1].x, v[2].x, v[3].x};
      const double bb[4] = {b01.x, b01.y, b23.x, b23.y};
      double fx[4];
      evo_cell_apply(*C, pc, bb, fx);
#pragma unroll
      for (int k = 0; k < 4; ++k) f[k] = make_double2(fx[k], 0.0);
    }
  }
  __device__ double2 di(int id) const { return __ldg(reinterpret_cast<const double2*>(dinv) + id); }
  static constexpr bool VY = true, AUX = true;  // (ux, uy) per node, d as the aux value
};

__device__ __forceinline__ double2 mask2(double2 v, double2 di) {
  return make_double2(di.x != 0.0 ? v.x : 0.0, di.y != 0.0 ? v.y : 0.0);
}

struct FineResid : FineBase {  // x = omega D^-1 r (pre-smoothing from zero), t = r - A x
  double om;
  const double* r;
  double* t;
  struct Raw {
    double2 dv, bv;
    double d;
  };
  __device__ void fetch(int id, int, int, bool, Raw& w) const {
    w.dv = di(id);
    w.bv = d2ldcg(r, id);
    w.d = __ldg(d + id);
  }
  __device__ double2 finish(const Raw& w, int, int, int, bool, double& aux) const {
    aux = w.d;
    return make_double2(om * w.dv.x * w.bv.x, om * w.dv.y * w.bv.y);
  }
  __device__ double2 in(int id, int i, int j, bool dup, double& aux) const {
    aux = 0.0;
    if (id < 0) return make_double2(0.0, 0.0);
    Raw w;
    fetch(id, i, j, dup, w);
    return finish(w, id, i, j, dup, aux);
  }
  struct ORaw {
    double2 bv, dv;
  };
  __device__ void ofetch(int id, ORaw& o) const {
    o.bv = d2ldcg(r, id);
    o.dv = di(id);
  }
  __device__ void outp(int id, double2 Av, double2, const ORaw& o) const {
    d2st(t, id, mask2(make_double2(o.bv.x - Av.x, o.bv.y - Av.y), o.dv));
  }
  __device__ void out(int id, double2 Av, double2 v) const {
    ORaw o;
    ofetch(id, o);
    outp(id, Av, v, o);
  }
};

// ---- global loads of the coarse-level kernels: every input of a kernel was written by an
// earlier kernel, so the read-only / L1 path is coherent
struct GMem {
  __device__ static double2 v2(const double* p, int i) {
    return __ldg(reinterpret_cast<const double2*>(p) + i);
  }
  __device__ static int4 row(const int4* p, int j) { return __ldg(p + j); }
};

// node id in a row entry (lo, hi, start); up: the slit row's duplicates as seen from above
__device__ __forceinline__ int mg_row_node(const DMesh& m, int4 rw, int i, int j, bool up) {
  if (i < rw.x || i >= rw.y) return -1;
  if (up && j == m.notch_row && i >= m.notch_lo && i < m.notch_hi)
    return m.dup_start + (i - m.notch_lo);
  return rw.z + (i - rw.x);
}

// prolongation (P e_{l+1}) at node (i, j) of level l; dup = upper-face slit node
template <class MC>
__device__ __forceinline__ double2 mg_prolong(const DMesh& mf, const DMesh& mc,
                                              const double* ec, int i, int j, bool dup) {
  const bool up = dup || (mf.notch_row >= 0 && j > mf.notch_row);
  const int I0 = i >> 1, J0 = j >> 1, I1 = I0 + (i & 1), J1 = J0 + (j & 1);
  const double w = ((i & 1) ? 0.5 : 1.0) * ((j & 1) ? 0.5 : 1.0);
  const int4 r0 = MC::row(mc.nrow, J0), r1 = MC::row(mc.nrow, min(J1, mc.ny));
  const int c00 = mg_row_node(mc, r0, I0, J0, up), c10 = mg_row_node(mc, r0, I1, J0, up);
  const int c01 = mg_row_node(mc, r1, I0, J1, up), c11 = mg_row_node(mc, r1, I1, J1, up);
  const double2 v00 = MC::v2(ec, max(c00, 0)), v10 = MC::v2(ec, max(c10, 0));
  const double2 v01 = MC::v2(ec, max(c01, 0)), v11 = MC::v2(ec, max(c11, 0));
  // distinct corners only (I1 == I0 / J1 == J0 on even positions)
  const double a00 = c00 >= 0 ? w : 0.0;
  const double a10 = (c10 >= 0 && I1 != I0) ? w : 0.0;
  const double a01 = (c01 >= 0 && J1 != J0) ? w : 0.0;
  const double a11 = (c11 >= 0 && I1 != I0 && J1 != J0) ? w : 0.0;
  return make_double2(a00 * v00.x + a10 * v10.x + a01 * v01.x + a11 * v11.x,
                      a00 * v00.y + a10 * v10.y + a01 * v01.y + a11 * v11.y);
}

// The bilinear prolongation of a fine-level march.  A lane keeps its fine column i, so its
// coarse sources are the fixed columns I0 = i/2, I1 = I0 + (i odd) of coarse rows J0 = j/2,
// J1 = J0 + (j odd).  The march visits the node rows in order (fetch(j) one row step ahead of
// finish(j), fetch(j + 1) after finish(j)), so the lane holds exactly two coarse rows -- lo = J0
// and hi = J0 + 1 -- and moves them by the parity of j: an odd row loads its hi row (one row-
// table entry and two values per TWO fine rows), an even row takes lo <- hi.  The slit's faces
// differ only on the coarse slit row, reloaded once when the march passes the fine slit row.
// A lane whose rows are not consecutive (first row of a unit, holes of an L-panel) starts over.
// Same products and order as mg_prolong: a00 v00 + a10 v10 + a01 v01 + a11 v11.
template <class V>
struct ProlongMarch {
  int last_j = -0x4000;
  V l0, l1, h0, h1;
  __device__ static V zero();
  __device__ static V load(const double* e, int c);
  __device__ static V comb(double a0, V v0, double a1, V v1, double a2, V v2, double a3, V v3);
  __device__ static void row(const DMesh& mc, const double* ec, int J, bool up, int I0, int I1,
                             V& v0, V& v1) {
    const int4 rw = __ldg(mc.nrow + min(J, mc.ny));
    const int c0 = mg_row_node(mc, rw, I0, J, up);
    const int c1 = I1 != I0 ? mg_row_node(mc, rw, I1, J, up) : -1;
    v0 = c0 >= 0 ? load(ec, c0) : zero();
    v1 = c1 >= 0 ? load(ec, c1) : zero();
  }
  // the loads of node row j (not a duplicate), one row step ahead of value(i, j)
  __device__ void fetch(const DMesh& mf, const DMesh& mc, const double* ec, int i, int j) {
    const int R = mf.notch_row;
    const bool up = R >= 0 && j > R;
    const int I0 = i >> 1, I1 = I0 + (i & 1), J0 = j >> 1;
    if (j != last_j + 1) {
      row(mc, ec, J0, up, I0, I1, l0, l1);
      h0 = h1 = zero();
      if (j & 1) row(mc, ec, J0 + 1, up, I0, I1, h0, h1);
    } else {
      if (j & 1) {
        row(mc, ec, J0 + 1, up, I0, I1, h0, h1);
      } else {
        l0 = h0;
        l1 = h1;
      }
      if (j == R + 1 && R >= 0) row(mc, ec, J0, true, I0, I1, l0, l1);
    }
    last_j = j;
  }
  __device__ V value(int i, int j) const {
    const double w = ((i & 1) ? 0.5 : 1.0) * ((j & 1) ? 0.5 : 1.0);
    const double a10 = (i & 1) ? w : 0.0, a01 = (j & 1) ? w : 0.0;
    const double a11 = ((i & 1) && (j & 1)) ? w : 0.0;
    return comb(w, l0, a10, l1, a01, h0, a11, h1);
  }
  // stateless (the row below a unit, the slit's upper face): four direct loads
  __device__ static V direct(const DMesh& mf, const DMesh& mc, const double* ec, int i, int j,
                             bool dup) {
    const bool up = dup || (mf.notch_row >= 0 && j > mf.notch_row);
    const int I0 = i >> 1, I1 = I0 + (i & 1), J0 = j >> 1;
    V a0, a1, b0 = zero(), b1 = zero();
    row(mc, ec, J0, up, I0, I1, a0, a1);
    if (j & 1) row(mc, ec, J0 + 1, up, I0, I1, b0, b1);
    const double w = ((i & 1) ? 0.5 : 1.0) * ((j & 1) ? 0.5 : 1.0);
    const double a10 = (i & 1) ? w : 0.0, a01 = (j & 1) ? w : 0.0;
    const double a11 = ((i & 1) && (j & 1)) ? w : 0.0;
    return comb(w, a0, a10, a1, a01, b0, a11, b1);
  }
};
template <> __device__ __forceinline__ double ProlongMarch<double>::zero() { return 0.0; }
template <> __device__ __forceinline__ double ProlongMarch<double>::load(const double* e, int c) {
  return __ldg(e + c);
}
template <> __device__ __forceinline__ double ProlongMarch<double>::comb(
    double a0, double v0, double a1, double v1, double a2, double v2, double a3, double v3) {
  return a0 * v0 + a1 * v1 + a2 * v2 + a3 * v3;
}
template <> __device__ __forceinline__ double2 ProlongMarch<double2>::zero() {
  return make_double2(0.0, 0.0);
}
template <> __device__ __forceinline__ double2 ProlongMarch<double2>::load(const double* e, int c) {
  return __ldg(reinterpret_cast<const double2*>(e) + c);
}
template <> __device__ __forceinline__ double2 ProlongMarch<double2>::comb(
    double a0, double2 v0, double a1, double2 v1, double a2, double2 v2, double a3, double2 v3) {
  return make_double2(a0 * v0.x + a1 * v1.x + a2 * v2.x + a3 * v3.x,
                      a0 * v0.y + a1 * v1.y + a2 * v2.y + a3 * v3.y);
}

struct FineSmooth : FineBase {  // y = omega D^-1 r + P e_1, z = y + omega D^-1 (r - A y); r.z
  double om;
  const double* r;
  double* z;
  const DMesh* mf;
  const DMesh* mc;
  const double* ec;
  double* rz;
  mutable ProlongMarch<double2> pm;  // the level-1 corrections of the bilinear prolongation
  struct Raw {
    double2 dv, bv;
    double d;
  };
  __device__ void fetch(int id, int i, int j, bool, Raw& w) const {
    w.dv = di(id);
    w.bv = d2ldcg(r, id);
    w.d = __ldg(d + id);
    pm.fetch(*mf, *mc, ec, i, j);
  }
  __device__ double2 smooth0(const Raw& w, double2 pe) const {
    return mask2(make_double2(om * w.dv.x * w.bv.x + pe.x, om * w.dv.y * w.bv.y + pe.y), w.dv);
  }
  __device__ double2 finish(const Raw& w, int, int i, int j, bool, double& aux) const {
    aux = w.d;
    return smooth0(w, pm.value(i, j));
  }
  __device__ double2 in(int id, int i, int j, bool dup, double& aux) const {
    aux = 0.0;
    if (id < 0) return make_double2(0.0, 0.0);
    Raw w;
    w.dv = di(id);
    w.bv = d2ldcg(r, id);
    aux = __ldg(d + id);
    return smooth0(w, ProlongMarch<double2>::direct(*mf, *mc, ec, i, j, dup));
  }
  __device__ void out2(int id, double2 Av, double2 y, double2 dv, double2 bv) const {
    const double2 ev = make_double2(y.x + om * dv.x * (bv.x - Av.x),
                                    y.y + om * dv.y * (bv.y - Av.y));
    d2st(z, id, ev);
    *rz += bv.x * ev.x + bv.y * ev.y;
  }
#if PFB_SMOOTH_OPRE
  struct ORaw {
    double2 bv, dv;
  };
  __device__ void ofetch(int id, ORaw& o) const {
    o.bv = d2ldcg(r, id);
    o.dv = di(id);
  }
  __device__ void outp(int id, double2 Av, double2 y, const ORaw& o) const {
    out2(id, Av, y, o.dv, o.bv);
  }
#endif
  __device__ void out(int id, double2 Av, double2 y) const {
    out2(id, Av, y, di(id), d2ldcg(r, id));
  }
};

struct FineWarm : FineBase {  // q_k = A u_k (masked); u_j.q_k (j <= k), u_k.b (b = r on entry)
  const double* u;
  double* qk;
  const double* uj[MG_WARM];
  int k;
  const double* b;
  double* acc;  // [MG_WARM + 2]: u_0.q_k .. u_k.q_k, u_k.b, b.b
  struct Raw {
    double2 uv, dv;
    double d;
  };
  __device__ void fetch(int id, int, int, bool, Raw& w) const {
    w.uv = __ldg(reinterpret_cast<const double2*>(u) + id);
    w.dv = di(id);
    w.d = __ldg(d + id);
  }
  __device__ double2 finish(const Raw& w, int, int, int, bool, double& aux) const {
    aux = w.d;
    return mask2(w.uv, w.dv);
  }
  __device__ double2 in(int id, int i, int j, bool dup, double& aux) const {
    aux = 0.0;
    if (id < 0) return make_double2(0.0, 0.0);
    Raw w;
    fetch(id, i, j, dup, w);
    return finish(w, id, i, j, dup, aux);
  }
  __device__ void out(int id, double2 Av, double2 uv) const {
    const double2 qv = mask2(Av, di(id));
    d2st(qk, id, qv);
#pragma unroll
    for (int j = 0; j < MG_WARM; ++j) {
      if (j > k) break;
      const double2 a = j == k ? uv : mask2(__ldg(reinterpret_cast<const double2*>(uj[j]) + id), di(id));
      acc[j] += a.x * qv.x + a.y * qv.y;
    }
    const double2 bv = __ldg(reinterpret_cast<const double2*>(b) + id);
    acc[MG_WARM] += uv.x * bv.x + uv.y * bv.y;
    if (k == 0) acc[MG_WARM + 1] += bv.x * bv.x + bv.y * bv.y;
  }
};

__device__ __forceinline__ double mg_hash01(unsigned k) {
  k ^= k >> 16; k *= 0x7feb352du; k ^= k >> 15; k *= 0x846ca68bu; k ^= k >> 16;
  return (double)(k & 0xffffff) * (1.0 / 16777216.0) - 0.5;
}

struct FinePow : FineBase {  // power step vout = D^-1 A vin (vin == nullptr: hashed start)
  const double* vin;
  double* vout;
  struct Raw {
    double2 v, dv;
    double d;
  };
  __device__ void fetch(int id, int, int, bool, Raw& w) const {
    w.v = vin ? d2ldcg(vin, id) : make_double2(mg_hash01(2u * id + 1u), mg_hash01(2u * id + 2u));
    w.dv = di(id);
    w.d = __ldg(d + id);
  }
  __device__ double2 finish(const Raw& w, int, int, int, bool, double& aux) const {
    aux = w.d;
    return mask2(w.v, w.dv);
  }
  __device__ double2 in(int id, int i, int j, bool dup, double& aux) const {
    aux = 0.0;
    if (id < 0) return make_double2(0.0, 0.0);
    Raw w;
    fetch(id, i, j, dup, w);
    return finish(w, id, i, j, dup, aux);
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
  const DMesh* own = nullptr;  // row strips: p.q over owned nodes only (pf_mgd.cuh)
  struct Raw {
    double2 zv, po;
    double d;
  };
  __device__ void fetch(int id, int, int, bool, Raw& w) const {
    w.zv = d2ldcg(z, id);
    w.po = pold ? d2ldcg(pold, id) : make_double2(0.0, 0.0);
    w.d = __ldg(d + id);
  }
  __device__ double2 finish(const Raw& w, int, int, int, bool, double& aux) const {
    aux = w.d;
    if (!pold) return w.zv;
    return make_double2(w.zv.x + beta * w.po.x, w.zv.y + beta * w.po.y);
  }
  __device__ double2 in(int id, int i, int j, bool dup, double& aux) const {
    aux = 0.0;
    if (id < 0) return make_double2(0.0, 0.0);
    Raw w;
    fetch(id, i, j, dup, w);
    return finish(w, id, i, j, dup, aux);
  }
  __device__ void out2(int id, double2 Av, double2 p, double2 dv) const {
    const double2 qv = mask2(Av, dv);
    d2st(pnew, id, p);
    d2st(q, id, qv);
    if (!own || node_owned(*own, id)) *pq += p.x * qv.x + p.y * qv.y;
  }
  struct ORaw {
    double2 dv;
  };
  __device__ void ofetch(int id, ORaw& o) const { o.dv = di(id); }
  __device__ void outp(int id, double2 Av, double2 p, const ORaw& o) const { out2(id, Av, p, o.dv); }
  __device__ void out(int id, double2 Av, double2 p) const { out2(id, Av, p, di(id)); }
};

// ---- coarse levels: node-parallel phases ----------------------------------------------------
// Visit every node of a level: items are (node row or the slit-duplicate row, 32-column chunk);
// f(id, i, j, dup) per existing node.  worker/nw count warps.
template <class M, class F>
__device__ __forceinline__ void mg_for_nodes(const DMesh& m, int worker, int nw, F&& f) {
  const int lane = threadIdx.x & 31;
  const int chunks = (m.nx + 1 + 31) / 32;
  const int rows = m.ny + 1 + (m.notch_row >= 0 ? 1 : 0);
  for (int it = worker; it < rows * chunks; it += nw) {
    const int row = it / chunks, i = (it % chunks) * 32 + lane;
    if (row <= m.ny) {
      const int id = mg_row_node(m, M::row(m.nrow, row), i, row, false);
      if (id >= 0) f(id, i, row, false);
    } else if (i >= m.notch_lo && i < m.notch_hi) {
      f(m.dup_start + (i - m.notch_lo), i, m.notch_row, true);
    }
  }
}
__host__ __device__ inline int mg_items(int nx, int ny, bool notch) {
  return (ny + 1 + (notch ? 1 : 0)) * ((nx + 1 + 31) / 32);
}

// ---- coarse levels in assembled form: one thread per node, slot-major index and stencil
// arrays, every load independent (two dependent rounds: indices, then values) -------------------
__device__ __forceinline__ double mg_rw(int s) {  // restriction weight of slot s
  const int a = s < 9 ? s % 3 - 1 : s - 10, b = s < 9 ? s / 3 - 1 : 0;
  return (a ? 0.5 : 1.0) * (b ? 0.5 : 1.0);
}
// Node-parallel kernels of the assembled form: a half-warp per node, one lane per stencil /
// restriction / prolongation slot, so every index and value load of a node is in flight at
// once (two dependent rounds); the half-warp sum is a fixed butterfly (bit-reproducible).
template <int W = 16>
__device__ __forceinline__ double2 hw_sum(double2 v) {  // butterfly over W aligned lanes
#pragma unroll
  for (int o = W / 2; o > 0; o >>= 1) {
    v.x += __shfl_xor_sync(0xffffffffu, v.x, o);
    v.y += __shfl_xor_sync(0xffffffffu, v.y, o);
  }
  return v;
}
// The 2x2 block of slot s2 at node id.  The grid-level kernels read it in FP32 (MgLevel::s32,
// default; PFB200_MG_S32=0 at handle creation: FP64): the V-cycle is only the preconditioner --
// the PCG's operator, residual and stopping test stay FP64 -- and the coarse levels' stencil
// products are bound by these loads.  tests/test_gpu_mg.py compares both on cracked states.
__device__ __forceinline__ void mg_s4(const MgLevel& L, int n, int id, int s2, double& sxx,
                                      double& sxy, double& syx, double& syy) {
  if (L.s32) {  // one 16-byte load per block: Sf is [MG_NS][n] float4 (xx, xy, yx, yy)
    const float4 b = __ldg(reinterpret_cast<const float4*>(L.Sf) + (size_t)s2 * n + id);
    sxx = b.x;
    if (L.scalar) {  // the packed scalar field: xy, yx, yy are exactly zero (warp-uniform)
      sxy = syx = syy = 0.0;
      return;
    }
    sxy = b.y;
    syx = b.z;
    syy = b.w;
    return;
  }
  const double* Sp = L.S + (size_t)(4 * s2) * n + id;
  sxx = __ldg(Sp);
  if (L.scalar) {
    sxy = syx = syy = 0.0;
    return;
  }
  sxy = __ldg(Sp + n);
  syx = __ldg(Sp + 2 * (size_t)n);
  syy = __ldg(Sp + 3 * (size_t)n);
}
// slot s2 of S_s x[nbr_s] at node id (zero for s2 >= MG_NS or no coupling)
template <class X>
__device__ __forceinline__ double2 mg_slot_apply(const MgLevel& L, int n, int id, int s2,
                                                 X&& xval) {
  if (s2 >= MG_NS || id >= n) return make_double2(0.0, 0.0);
  const int k = __ldg(L.nbr + (size_t)s2 * n + id);
  if (k < 0) return make_double2(0.0, 0.0);
  double sxx, sxy, syx, syy;
  mg_s4(L, n, id, s2, sxx, sxy, syx, syy);
  const double2 x = xval(k);
  return make_double2(sxx * x.x + sxy * x.y, syx * x.x + syy * x.y);
}
// LPN lanes per node (16: small levels, every load of a node in flight at once; 4 / 1: larger
// levels, latency hidden by the many resident warps).  Slot partial sums are combined in a
// fixed order either way (bit-reproducible).
template <int LPN>
struct NodeMap {
  __device__ static int lane() { return LPN == 1 ? 0 : (int)(threadIdx.x & (LPN - 1)); }
  __device__ static int first() { return (int)((blockIdx.x * blockDim.x + threadIdx.x) / LPN); }
  __device__ static int stride() { return (int)((gridDim.x * blockDim.x) / LPN); }
  __device__ static int end(int n) {  // warp-uniform trip counts (32 / LPN nodes per warp)
    return LPN == 1 ? n : ((n + 32 / LPN - 1) / (32 / LPN)) * (32 / LPN);
  }
  __device__ static double2 sum(double2 v) { return LPN == 1 ? v : hw_sum<LPN>(v); }
};
template <int LPN, class X>
__device__ __forceinline__ double2 mg_apply(const MgLevel& L, int n, int id, X&& xval) {
  double2 acc = make_double2(0.0, 0.0);
#pragma unroll
  for (int s2 = NodeMap<LPN>::lane(); s2 < MG_NS; s2 += LPN) {
    const double2 v = mg_slot_apply(L, n, id, s2, xval);
    acc.x += v.x;
    acc.y += v.y;
  }
  return NodeMap<LPN>::sum(acc);
}
#define MG_FOR_NODE_L(n) \
  for (int id = NodeMap<LPN>::first(); id < NodeMap<LPN>::end(n); id += NodeMap<LPN>::stride())
#define MG_LEAD (NodeMap<LPN>::lane() == 0 && id < n)

// restriction b = P^T t_{l-1} (masked at dead dofs)
template <int LPN>
__global__ void __launch_bounds__(MG_NT) k_mg_srestrict(MgArgs A, int l) {
  const MgLevel& L = A.L[l];
  const int n = L.m.n_nodes;
  const double* tf = A.L[l - 1].t;
  MG_FOR_NODE_L(n) {
    double2 v = make_double2(0.0, 0.0);
    if (id < n) {
#pragma unroll
      for (int s2 = NodeMap<LPN>::lane(); s2 < 12; s2 += LPN) {
        const int f = __ldg(L.rid + (size_t)s2 * n + id);
        if (f >= 0) {
          const double2 t = GMem::v2(tf, f);
          const double w = mg_rw(s2);
          v.x += w * t.x;
          v.y += w * t.y;
        }
      }
    }
    v = NodeMap<LPN>::sum(v);
    if (MG_LEAD) d2st(L.b, id, mask2(v, GMem::v2(L.dinv, id)));
  }
}
// t = b - A x, x = omega D^-1 b
template <int LPN>
__global__ void __launch_bounds__(MG_NT) k_mg_sresid(MgArgs A, int l) {
  const MgLevel& L = A.L[l];
  const int n = L.m.n_nodes;
  const double om = __ldcg(&A.ctl->omega[l]);
  MG_FOR_NODE_L(n) {
    const double2 Av = mg_apply<LPN>(L, n, id, [&](int k) -> double2 {
      const double2 di = GMem::v2(L.dinv, k), bv = GMem::v2(L.b, k);
      return make_double2(om * di.x * bv.x, om * di.y * bv.y);
    });
    if (MG_LEAD) {
      const double2 di = GMem::v2(L.dinv, id), bv = GMem::v2(L.b, id);
      d2st(L.t, id, mask2(make_double2(bv.x - Av.x, bv.y - Av.y), di));
    }
  }
}
// y = omega D^-1 b + P e_{l+1} (into t)
template <int LPN>
__global__ void __launch_bounds__(MG_NT) k_mg_sprolongate(MgArgs A, int l) {
  const MgLevel& L = A.L[l];
  const int n = L.m.n_nodes;
  const double om = __ldcg(&A.ctl->omega[l]);
  const double* ec = A.L[l + 1].e;
  MG_FOR_NODE_L(n) {
    double2 v = make_double2(0.0, 0.0), cnt = make_double2(0.0, 0.0);
    if (id < n) {
#pragma unroll
      for (int s2 = NodeMap<LPN>::lane(); s2 < 4; s2 += LPN) {
        const int c = __ldg(L.pid + (size_t)s2 * n + id);
        if (c >= 0) {
          const double2 e = GMem::v2(ec, c);
          v.x += e.x;
          v.y += e.y;
          cnt.x += 1.0;
        }
      }
    }
    v = NodeMap<LPN>::sum(v);
    cnt = NodeMap<LPN>::sum(cnt);
    if (MG_LEAD) {
      const double w = 1.0 / cnt.x;  // bilinear weights: 1, 1/2 or 1/4 (distinct sources)
      const double2 di = GMem::v2(L.dinv, id), bv = GMem::v2(L.b, id);
      d2st(L.t, id, mask2(make_double2(om * di.x * bv.x + w * v.x, om * di.y * bv.y + w * v.y), di));
    }
  }
}
// e = y + omega D^-1 (b - A y), y in t
template <int LPN>
__global__ void __launch_bounds__(MG_NT) k_mg_ssmooth(MgArgs A, int l) {
  const MgLevel& L = A.L[l];
  const int n = L.m.n_nodes;
  const double om = __ldcg(&A.ctl->omega[l]);
  MG_FOR_NODE_L(n) {
    const double2 Ay = mg_apply<LPN>(L, n, id, [&](int k) -> double2 { return GMem::v2(L.t, k); });
    if (MG_LEAD) {
      const double2 y = GMem::v2(L.t, id), di = GMem::v2(L.dinv, id), bv = GMem::v2(L.b, id);
      d2st(L.e, id, make_double2(y.x + om * di.x * (bv.x - Ay.x), y.y + om * di.y * (bv.y - Ay.y)));
    }
  }
}
// Fused down-sweep of a small level (one lane per stencil slot): the restriction of t_{l-1} is
// evaluated at each neighbour by the lane that multiplies it (12 source loads per lane, all in
// flight), x = omega D^-1 b, t = b - A x; b is stored for the up-sweep.  Saves the separate
// restriction kernel's launch and dependent rounds.
template <int LPN>
__global__ void __launch_bounds__(MG_NT) k_mg_sdown(MgArgs A, int l) {
  const MgLevel& L = A.L[l];
  const int n = L.m.n_nodes;
  const double om = __ldcg(&A.ctl->omega[l]);
  const double* tf = A.L[l - 1].t;
  MG_FOR_NODE_L(n) {
    double2 acc = make_double2(0.0, 0.0), bc = make_double2(0.0, 0.0);
    if (id < n) {
#pragma unroll
      for (int s2 = NodeMap<LPN>::lane(); s2 < MG_NS; s2 += LPN) {
        const int k = __ldg(L.nbr + (size_t)s2 * n + id);
        if (k < 0) continue;
        int f[12];
#pragma unroll
        for (int j = 0; j < 12; ++j) f[j] = __ldg(L.rid + (size_t)j * n + k);
        double2 b = make_double2(0.0, 0.0);
#pragma unroll
        for (int j = 0; j < 12; ++j) {
          if (f[j] < 0) continue;
          const double2 t = GMem::v2(tf, f[j]);
          const double w = mg_rw(j);
          b.x += w * t.x;
          b.y += w * t.y;
        }
        const double2 di = GMem::v2(L.dinv, k);
        b = mask2(b, di);
        if (s2 == 4) bc = b;  // the node itself
        double sxx, sxy, syx, syy;
        mg_s4(L, n, id, s2, sxx, sxy, syx, syy);
        const double2 x = make_double2(om * di.x * b.x, om * di.y * b.y);
        acc.x += sxx * x.x + sxy * x.y;
        acc.y += syx * x.x + syy * x.y;
      }
    }
    acc = NodeMap<LPN>::sum(acc);
    bc = NodeMap<LPN>::sum(bc);
    if (MG_LEAD) {
      d2st(L.b, id, bc);
      d2st(L.t, id, mask2(make_double2(bc.x - acc.x, bc.y - acc.y), GMem::v2(L.dinv, id)));
    }
  }
}
// Fused up-sweep of a small level: y = omega D^-1 b + P e_{l+1} evaluated at each neighbour by
// its lane, e = y + omega D^-1 (b - A y)
template <int LPN>
__global__ void __launch_bounds__(MG_NT) k_mg_sup(MgArgs A, int l) {
  const MgLevel& L = A.L[l];
  const int n = L.m.n_nodes;
  const double om = __ldcg(&A.ctl->omega[l]);
  const double* ec = A.L[l + 1].e;
  MG_FOR_NODE_L(n) {
    double2 acc = make_double2(0.0, 0.0), yc = make_double2(0.0, 0.0);
    if (id < n) {
#pragma unroll
      for (int s2 = NodeMap<LPN>::lane(); s2 < MG_NS; s2 += LPN) {
        const int k = __ldg(L.nbr + (size_t)s2 * n + id);
        if (k < 0) continue;
        int c[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) c[j] = __ldg(L.pid + (size_t)j * n + k);
        const double w = 1.0 / ((c[0] >= 0) + (c[1] >= 0) + (c[2] >= 0) + (c[3] >= 0));
        double2 pe = make_double2(0.0, 0.0);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          if (c[j] < 0) continue;
          const double2 e = GMem::v2(ec, c[j]);
          pe.x += e.x;
          pe.y += e.y;
        }
        const double2 di = GMem::v2(L.dinv, k), bv = GMem::v2(L.b, k);
        const double2 y = mask2(make_double2(om * di.x * bv.x + w * pe.x, om * di.y * bv.y + w * pe.y), di);
        if (s2 == 4) yc = y;
        double sxx, sxy, syx, syy;
        mg_s4(L, n, id, s2, sxx, sxy, syx, syy);
        acc.x += sxx * y.x + sxy * y.y;
        acc.y += syx * y.x + syy * y.y;
      }
    }
    acc = NodeMap<LPN>::sum(acc);
    yc = NodeMap<LPN>::sum(yc);
    if (MG_LEAD) {
      const double2 di = GMem::v2(L.dinv, id), bv = GMem::v2(L.b, id);
      d2st(L.e, id, make_double2(yc.x + om * di.x * (bv.x - acc.x), yc.y + om * di.y * (bv.y - acc.y)));
    }
  }
}
// ---- large coarse levels (>= 2^20 nodes: on smaller, L2-resident levels the table kernels are
// faster, cfg2's 66 k-node level 1 125 vs 112 us per V-cycle), one thread per node over (row,
// 32-column chunk) items: neighbour /
// restriction / prolongation ids from the row tables where the stencil is regular (as
// pf_mgs.cuh's k_mgs_r*: the same products in the same order as the table kernels, bitwise
// equal; 40 B per node less index traffic per stencil product, 48 B per restriction)
__device__ __forceinline__ bool mg_regular(const DMesh& m, int i, int j, int4 rw) {
  if (j <= 0 || j >= m.ny || i <= rw.x || i >= rw.y - 1) return false;
  if (m.notch_row >= 0 && j >= m.notch_row - 1 && j <= m.notch_row + 1) return false;
  const int4 a = __ldg(m.nrow + j - 1), b = __ldg(m.nrow + j + 1);
  return a.x == rw.x && a.y == rw.y && b.x == rw.x && b.y == rw.y;
}
template <class X>
__device__ __forceinline__ double2 mg_row_apply(const MgLevel& L, int n, int id, int i, int j,
                                                bool dup, X&& xval) {
  double2 acc = make_double2(0.0, 0.0);
  const int4 rw = __ldg(L.m.nrow + j);
  if (!dup && mg_regular(L.m, i, j, rw)) {
    const int len = rw.y - rw.x;
#pragma unroll
    for (int s2 = 0; s2 < 9; ++s2) {
      const int k = id + (s2 / 3 - 1) * len + (s2 % 3 - 1);
      double sxx, sxy, syx, syy;
      mg_s4(L, n, id, s2, sxx, sxy, syx, syy);
      const double2 x = xval(k);
      acc.x += sxx * x.x + sxy * x.y;
      acc.y += syx * x.x + syy * x.y;
    }
  } else {
#pragma unroll
    for (int s2 = 0; s2 < MG_NS; ++s2) {
      const double2 v = mg_slot_apply(L, n, id, s2, xval);
      acc.x += v.x;
      acc.y += v.y;
    }
  }
  return acc;
}
__global__ void __launch_bounds__(MG_NT) k_mg_rrestrict(MgArgs A, int l) {
  const MgLevel& L = A.L[l];
  const DMesh& mf = A.L[l - 1].m;
  const int n = L.m.n_nodes;
  const double* tf = A.L[l - 1].t;
  mg_for_nodes<GMem>(L.m, (int)(blockIdx.x * MG_WARPS + (threadIdx.x >> 5)), (int)(gridDim.x * MG_WARPS), [&](int id, int I, int J, bool dup) {
    double2 v = make_double2(0.0, 0.0);
    const int j0 = 2 * J, i0 = 2 * I;
    bool reg = !dup && j0 >= 1 && j0 < mf.ny &&
               !(mf.notch_row >= 0 && j0 >= mf.notch_row - 1 && j0 <= mf.notch_row + 1);
    int4 r0 = make_int4(0, 0, 0, 0), rm = r0, rp = r0;
    if (reg) {
      r0 = __ldg(mf.nrow + j0);
      rm = __ldg(mf.nrow + j0 - 1);
      rp = __ldg(mf.nrow + j0 + 1);
      reg = rm.x == r0.x && rm.y == r0.y && rp.x == r0.x && rp.y == r0.y && i0 - 1 >= r0.x &&
            i0 + 1 <= r0.y - 1;
    }
    if (reg) {
      const int st[3] = {rm.z, r0.z, rp.z};
#pragma unroll
      for (int s2 = 0; s2 < 9; ++s2) {
        const double2 t = GMem::v2(tf, st[s2 / 3] + (i0 + (s2 % 3 - 1) - r0.x));
        const double w = mg_rw(s2);
        v.x += w * t.x;
        v.y += w * t.y;
      }
    } else {
#pragma unroll
      for (int s2 = 0; s2 < 12; ++s2) {
        const int f = __ldg(L.rid + (size_t)s2 * n + id);
        if (f >= 0) {
          const double2 t = GMem::v2(tf, f);
          const double w = mg_rw(s2);
          v.x += w * t.x;
          v.y += w * t.y;
        }
      }
    }
    d2st(L.b, id, mask2(v, GMem::v2(L.dinv, id)));
  });
}
__global__ void __launch_bounds__(MG_NT) k_mg_rresid(MgArgs A, int l) {
  const MgLevel& L = A.L[l];
  const int n = L.m.n_nodes;
  const double om = __ldcg(&A.ctl->omega[l]);
  mg_for_nodes<GMem>(L.m, (int)(blockIdx.x * MG_WARPS + (threadIdx.x >> 5)), (int)(gridDim.x * MG_WARPS), [&](int id, int i, int j, bool dup) {
    const double2 Av = mg_row_apply(L, n, id, i, j, dup, [&](int k) -> double2 {
      const double2 di = GMem::v2(L.dinv, k), bv = GMem::v2(L.b, k);
      return make_double2(om * di.x * bv.x, om * di.y * bv.y);
    });
    const double2 di = GMem::v2(L.dinv, id), bv = GMem::v2(L.b, id);
    d2st(L.t, id, mask2(make_double2(bv.x - Av.x, bv.y - Av.y), di));
  });
}
__global__ void __launch_bounds__(MG_NT) k_mg_rsmooth(MgArgs A, int l) {
  const MgLevel& L = A.L[l];
  const int n = L.m.n_nodes;
  const double om = __ldcg(&A.ctl->omega[l]);
  mg_for_nodes<GMem>(L.m, (int)(blockIdx.x * MG_WARPS + (threadIdx.x >> 5)), (int)(gridDim.x * MG_WARPS), [&](int id, int i, int j, bool dup) {
    const double2 Ay = mg_row_apply(L, n, id, i, j, dup, [&](int k) -> double2 { return GMem::v2(L.t, k); });
    const double2 y = GMem::v2(L.t, id), di = GMem::v2(L.dinv, id), bv = GMem::v2(L.b, id);
    d2st(L.e, id, make_double2(y.x + om * di.x * (bv.x - Ay.x), y.y + om * di.y * (bv.y - Ay.y)));
  });
}

// Jacobi sweep out = in + omega D^-1 (b - A in) (grid coarsest level)
template <int LPN>
__global__ void __launch_bounds__(MG_NT) k_mg_ssweep(MgArgs A, int l, const double* in,
                                                     double* out) {
  const MgLevel& L = A.L[l];
  const int n = L.m.n_nodes;
  const double om = __ldcg(&A.ctl->omega[l]);
  MG_FOR_NODE_L(n) {
    const double2 Ax = mg_apply<LPN>(L, n, id, [&](int k) -> double2 { return GMem::v2(in, k); });
    if (MG_LEAD) {
      const double2 x = GMem::v2(in, id), di = GMem::v2(L.dinv, id), bv = GMem::v2(L.b, id);
      d2st(out, id, make_double2(x.x + om * di.x * (bv.x - Ax.x), x.y + om * di.y * (bv.y - Ax.y)));
    }
  }
}
// power step at one node of a coarse level (half-warp per node; every lane of the warp must
// call it: id >= n makes the half-warp idle): vout = D^-1 A vin (vin == nullptr: hashed start)
template <int LPN>
__device__ __forceinline__ void mg_spow(const MgLevel& L, const double* vin, double* vout, int id) {
  const int n = L.m.n_nodes;
  double2 acc = make_double2(0.0, 0.0);
#pragma unroll
  for (int s2 = NodeMap<LPN>::lane(); s2 < MG_NS; s2 += LPN) {
    const double2 v = mg_slot_apply(L, n, id, s2, [&](int k) -> double2 {
      const double2 di = GMem::v2(L.dinv, k);
      const double2 x = vin ? GMem::v2(vin, k)
                            : make_double2(mg_hash01(2u * k + 1u), mg_hash01(2u * k + 2u));
      return mask2(x, di);
    });
    acc.x += v.x;
    acc.y += v.y;
  }
  const double2 Av = NodeMap<LPN>::sum(acc);
  if (NodeMap<LPN>::lane() == 0 && id < n) {
    const double2 di = GMem::v2(L.dinv, id);
    d2st(vout, id, make_double2(di.x * Av.x, di.y * Av.y));
  }
}
// setup: assemble the stencil of level l from its cell matrices, and its inverse diagonal
__global__ void __launch_bounds__(MG_NT) k_mg_stencil(MgArgs A, int l) {
  const MgLevel& L = A.L[l];
  const DMesh& m = L.m;
  const int n = m.n_nodes;
  mg_for_nodes<GMem>(m, blockIdx.x * MG_WARPS + (threadIdx.x >> 5), gridDim.x * MG_WARPS,
                     [&](int id, int i, int j, bool) {
    int nb[MG_NS];
#pragma unroll
    for (int s2 = 0; s2 < MG_NS; ++s2) nb[s2] = __ldg(L.nbr + (size_t)s2 * n + id);
    double acc[MG_NS][4];
#pragma unroll
    for (int s2 = 0; s2 < MG_NS; ++s2)
#pragma unroll
      for (int q = 0; q < 4; ++q) acc[s2][q] = 0.0;
    const int cdx[4] = {-1, 0, -1, 0}, cdy[4] = {-1, -1, 0, 0}, ck[4] = {2, 3, 1, 0};
#pragma unroll
    for (int c = 0; c < 4; ++c) {  // below-left, below-right, above-left, above-right
      const int ci = i + cdx[c], cj = j + cdy[c];
      const int e = mg_cell(m, ci, cj);
      if (e < 0) continue;
      int cn[4];
      cn[0] = mg_node(m, ci, cj, true);
      cn[1] = mg_node(m, ci + 1, cj, true);
      cn[2] = mg_node(m, ci + 1, cj + 1, false);
      cn[3] = mg_node(m, ci, cj + 1, false);
      const int k = ck[c];
      if (cn[k] != id) continue;  // the cell is on the other face of the slit
      const double* Ke = L.K + 64 * (size_t)e;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int qx = ci + ((q == 1 || q == 2) ? 1 : 0) - i, qy = cj + (q >= 2 ? 1 : 0) - j;
        int slot = qy < 0 ? 1 + qx : (qy > 0 ? 7 + qx : 4 + qx);
        if (qy == 0 && nb[slot] != cn[q]) slot = 9;
        const double kxx = __ldg(Ke + (2 * k) * 8 + 2 * q), kxy = __ldg(Ke + (2 * k) * 8 + 2 * q + 1);
        const double kyx = __ldg(Ke + (2 * k + 1) * 8 + 2 * q),
                     kyy = __ldg(Ke + (2 * k + 1) * 8 + 2 * q + 1);
#pragma unroll
        for (int s2 = 0; s2 < MG_NS; ++s2)
          if (s2 == slot) {
            acc[s2][0] += kxx; acc[s2][1] += kxy; acc[s2][2] += kyx; acc[s2][3] += kyy;
          }
      }
    }
#pragma unroll
    for (int s2 = 0; s2 < MG_NS; ++s2) {
#pragma unroll
      for (int q = 0; q < 4; ++q) L.S[(size_t)(4 * s2 + q) * n + id] = acc[s2][q];
      reinterpret_cast<float4*>(L.Sf)[(size_t)s2 * n + id] = make_float4(
          (float)acc[s2][0], (float)acc[s2][1], (float)acc[s2][2], (float)acc[s2][3]);
    }
    d2st(L.dinv, id, make_double2(acc[4][0] > 0.0 ? 1.0 / acc[4][0] : 0.0,
                                  acc[4][3] > 0.0 ? 1.0 / acc[4][3] : 0.0));
  });
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
    lane_ordered_sum<NV>(part, NV, nparts, s);
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
// warm start, step 1 (k = 0 .. MG_WARM-1): q_k = A u_k over the fine march, with the Gram
// partials u_j.q_k (j <= k), u_k.b and b.b; the guesses come from the mapped per-solve inputs
// (a kernel with k >= n_guess does nothing).  Partials: [CTA][MG_WARM * (MG_WARM + 1) / 2 + 4].
constexpr int MG_WP = MG_WARM * (MG_WARM + 1) / 2 + MG_WARM + 1;
__device__ __forceinline__ int mg_gidx(int j, int k) { return k * (k + 1) / 2 + j; }  // j <= k
__device__ __forceinline__ double* mg_warm_q(const MgArgs& A, int k) {
  return k == 0 ? A.L[0].t : (k == 1 ? A.z : A.q);
}
__global__ void __launch_bounds__(MG_NT, 2) k_mg_warm_q(MgArgs A, int k) {
  __shared__ MgWarp ws[MG_WARPS];
  __shared__ double red[MG_WARPS * (MG_WARM + 2)];
  const MgIn* in = A.in;
  if (k >= __ldg(&in->n_guess)) return;
  double acc[MG_WARM + 2];
#pragma unroll
  for (int j = 0; j < MG_WARM + 2; ++j) acc[j] = 0.0;
  FineWarm op{{&A.C, A.flags, A.d, A.L[0].dinv, A.phys, A.bq}, (const double*)in->guess[k], mg_warm_q(A, k),
              {(const double*)in->guess[0], (const double*)in->guess[1], (const double*)in->guess[2]},
              k, A.r, acc};
  const int w = blockIdx.x * MG_WARPS + (threadIdx.x >> 5);
  if (w < A.g0.n_units) mg_march(A.L[0].m, A.g0, w, op, ws[threadIdx.x >> 5]);
  mg_block_sum<MG_WARM + 2>(acc, red);
  if (threadIdx.x == 0) {
    double* p = A.part + (size_t)MG_WP * blockIdx.x;
#pragma unroll
    for (int j = 0; j < MG_WARM; ++j)
      if (j <= k) p[mg_gidx(j, k)] = acc[j];
    p[MG_WARM * (MG_WARM + 1) / 2 + k] = acc[MG_WARM];
    if (k == 0) p[MG_WP - 1] = acc[MG_WARM + 1];
  }
}

// solve init: x0 = U y with (U^T A U) y = U^T b (pivot-dropping Cholesky, identical in every
// CTA), r0 = b - sum y_k q_k; x0 = 0 without guesses.  ||b|| is the original right-hand side's
// (scipy: rtol * ||b||).  The last CTA sets the control block and the WHILE condition.
__global__ void __launch_bounds__(MG_NT) k_mg_init(MgArgs A, int n_wparts) {
  __shared__ double red[MG_WP];
  const MgIn* in = A.in;
  const int m = __ldg(&in->n_guess);
  double y[MG_WARM] = {0.0, 0.0, 0.0};
  double bb = -1.0;
  if (m > 0) {
    double g[MG_WP];
    mg_all_reduce<MG_WP>(A.part, n_wparts, red, g);
    bb = g[MG_WP - 1];
    double G[MG_WARM][MG_WARM], c[MG_WARM], L[MG_WARM][MG_WARM], z[MG_WARM];
    bool keep[MG_WARM];
#pragma unroll
    for (int i = 0; i < MG_WARM; ++i) {
      c[i] = i < m ? g[MG_WARM * (MG_WARM + 1) / 2 + i] : 0.0;
#pragma unroll
      for (int j = 0; j < MG_WARM; ++j) {
        G[i][j] = (i < m && j < m) ? g[mg_gidx(min(i, j), max(i, j))] : 0.0;
        L[i][j] = 0.0;
      }
    }
#pragma unroll
    for (int i = 0; i < MG_WARM; ++i) {
      double dd = G[i][i];
#pragma unroll
      for (int k = 0; k < i; ++k) dd -= L[i][k] * L[i][k];
      keep[i] = i < m && G[i][i] > 0.0 && dd > 1e-6 * G[i][i];
      const double lii = keep[i] ? sqrt(dd) : 1.0;
      L[i][i] = keep[i] ? lii : 0.0;
#pragma unroll
      for (int j = i + 1; j < MG_WARM; ++j) {
        double e = G[j][i];
#pragma unroll
        for (int k = 0; k < i; ++k) e -= L[j][k] * L[i][k];
        L[j][i] = keep[i] ? e / lii : 0.0;
      }
    }
#pragma unroll
    for (int i = 0; i < MG_WARM; ++i) {
      double e = c[i];
#pragma unroll
      for (int k = 0; k < i; ++k) e -= L[i][k] * z[k];
      z[i] = keep[i] ? e / L[i][i] : 0.0;
    }
#pragma unroll
    for (int i = MG_WARM - 1; i >= 0; --i) {
      double e = z[i];
#pragma unroll
      for (int k = i + 1; k < MG_WARM; ++k) e -= L[k][i] * y[k];
      y[i] = keep[i] ? e / L[i][i] : 0.0;
    }
  }
  double rr = 0.0;
  const double* u0 = m > 0 ? (const double*)in->guess[0] : nullptr;
  const double* u1 = m > 1 ? (const double*)in->guess[1] : nullptr;
  const double* u2 = m > 2 ? (const double*)in->guess[2] : nullptr;
  const double* q0 = mg_warm_q(A, 0);
  const double* q1 = mg_warm_q(A, 1);
  const double* q2 = mg_warm_q(A, 2);
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < A.ndof;
       i += (long long)gridDim.x * blockDim.x) {
    double rv = __ldcg(A.r + i), xv = 0.0;
    if (m > 0 && __ldg(A.L[0].dinv + i) != 0.0) {
      xv = y[0] * __ldg(u0 + i);
      rv -= y[0] * __ldcg(q0 + i);
      if (u1) { xv += y[1] * __ldg(u1 + i); rv -= y[1] * __ldcg(q1 + i); }
      if (u2) { xv += y[2] * __ldg(u2 + i); rv -= y[2] * __ldcg(q2 + i); }
      A.r[i] = rv;
    }
    A.x[i] = xv;
    rr += rv * rv;
  }
  double v[1] = {rr};
  if (mg_publish<1>(v, A.part + (size_t)MG_WP * n_wparts, &A.ctl->count, red)) {
    double tot[1];
    mg_all_reduce<1>(A.part + (size_t)MG_WP * n_wparts, gridDim.x, red, tot);
    if (threadIdx.x == 0) {
      MgCtl& c = *A.ctl;
      c.count = 0;
      c.rr = tot[0];
      c.maxiter = in->maxiter;
      c.target = in->target;
      c.bnorm = sqrt(m > 0 ? bb : tot[0]);
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
  FineResid op{{&A.C, A.flags, A.d, A.L[0].dinv, A.phys, A.bq}, om, A.r, A.L[0].t};
  const int w = blockIdx.x * MG_WARPS + (threadIdx.x >> 5);
  if (w < A.g0.n_units) mg_march(A.L[0].m, A.g0, w, op, ws[threadIdx.x >> 5]);
}

#define MG_GW (int)(blockIdx.x * MG_WARPS + (threadIdx.x >> 5)), (int)(gridDim.x * MG_WARPS)
// coarsest level on the grid (it does not fit the tail kernel's shared memory): dense inverse
// applied by one CTA, or Jacobi sweeps from zero (k_mg_jacobi0 then k_mg_ssweep ping-pong)
__global__ void __launch_bounds__(MG_NT) k_mg_coarse_dense(MgArgs A) {
  const MgLevel& L = A.L[A.n_levels - 1];
  const int nd = 2 * L.m.n_nodes;
  for (int i = threadIdx.x; i < nd; i += blockDim.x) {
    double s = 0.0;
    for (int j = 0; j < nd; ++j) s += __ldcg(A.Ainv + (size_t)i * nd + j) * __ldcg(L.b + j);
    L.e[i] = s;
  }
}
__global__ void __launch_bounds__(MG_NT) k_mg_jacobi0(MgArgs A, int l, double* out) {
  const MgLevel& L = A.L[l];
  const double om = __ldcg(&A.ctl->omega[l]);
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < 2LL * L.m.n_nodes;
       i += (long long)gridDim.x * blockDim.x)
    out[i] = om * __ldcg(L.dinv + i) * __ldcg(L.b + i);
}
// Tail: levels [n_tail, n_levels) in assembled form staged in dynamic shared memory
// (neighbour / restriction / prolongation tables, stencils, inverse diagonals, the dense
// coarsest inverse) and cycled by one CTA with CTA barriers, a half-warp per node: from the
// restriction of level n_tail - 1's residual (global) down to the coarsest solve and back up
// to e_{n_tail} (global).  Byte offsets come from the host (MgArgs::ts).
extern __shared__ __align__(16) unsigned char mg_tail_smem[];
struct TLevel {  // shared-memory view of one tail level
  int n;
  const int *nbr, *rid, *pid;
  const double *S, *dinv;
  double *b, *t, *e;
};
__device__ __forceinline__ TLevel mg_tl(const MgArgs& A, int l) {
  unsigned char* sm = mg_tail_smem;
  const MgTailSlot& o = A.ts[l];
  TLevel v;
  v.n = A.L[l].m.n_nodes;
  v.nbr = reinterpret_cast<const int*>(sm + o.nbr);
  v.rid = reinterpret_cast<const int*>(sm + o.rid);
  v.pid = reinterpret_cast<const int*>(sm + o.pid);
  v.S = reinterpret_cast<const double*>(sm + o.S);
  v.dinv = reinterpret_cast<const double*>(sm + o.dinv);
  v.b = reinterpret_cast<double*>(sm + o.b);
  v.t = reinterpret_cast<double*>(sm + o.t);
  v.e = reinterpret_cast<double*>(sm + o.e);
  return v;
}
__device__ __forceinline__ double2 ts2(const double* p, int i) {
  return reinterpret_cast<const double2*>(p)[i];
}
// S x at node id of a tail level: 4 lanes per node, lane q takes slots q, q+4, q+8
template <class X>
__device__ __forceinline__ double2 mg_tapply(const TLevel& L, int id, X&& xval) {
  const int q = threadIdx.x & 3, n = L.n;
  double2 v = make_double2(0.0, 0.0);
  if (id < n) {
#pragma unroll
    for (int s2 = q; s2 < MG_NS; s2 += 4) {
      const int k = L.nbr[s2 * n + id];
      if (k >= 0) {
        const double* Sp = L.S + (4 * s2) * n + id;
        const double2 x = xval(k);
        v.x += Sp[0] * x.x + Sp[n] * x.y;
        v.y += Sp[2 * n] * x.x + Sp[3 * n] * x.y;
      }
    }
  }
  return hw_sum<4>(v);
}
#define MG_TAIL_NODES(n) \
  for (int id = threadIdx.x >> 2, _e = (((n) + 7) >> 3) << 3; id < _e; id += blockDim.x >> 2)
constexpr int MG_TAIL_PASS = MG_TAIL_NT / 4;  // nodes per pass

__global__ void __launch_bounds__(MG_TAIL_NT) k_mg_tail(MgArgs A) {
  const int nl = A.n_levels, l0 = A.n_tail, c = nl - 1;
  const int q = threadIdx.x & 3;
  int tk = 0;
  auto TCLK = [&]() {
    if (A.tclk && threadIdx.x == 0 && tk < 32) A.tclk[tk++] = clock64();
  };
  TCLK();
  const int nd = 2 * A.L[c].m.n_nodes;
  double* Ainv = reinterpret_cast<double*>(mg_tail_smem + A.ts_ainv);
  __shared__ __align__(8) unsigned long long bar;
  if (threadIdx.x == 0) {  // stage the tables and this hierarchy's operators with TMA bulk copies
    unsigned total = 0;
    for (int l = l0; l < nl; ++l) {
      const size_t n = A.L[l].m.n_nodes;
      total += mg_r16(4 * MG_NS * n) + mg_r16(4 * 12 * n) + (l < c ? mg_r16(4 * 4 * n) : 0) +
               mg_r16(8 * 4 * MG_NS * n) + mg_r16(16 * n);
    }
    if (A.dense) total += mg_r16(8 * (size_t)nd * nd);
    mg_mbar_init_expect(&bar, total);
    for (int l = l0; l < nl; ++l) {
      const TLevel v = mg_tl(A, l);
      const MgLevel& G = A.L[l];
      const size_t n = v.n;
      mg_bulk_g2s(v.nbr, G.nbr, mg_r16(4 * MG_NS * n), &bar);
      mg_bulk_g2s(v.rid, G.rid, mg_r16(4 * 12 * n), &bar);
      if (l < c) mg_bulk_g2s(v.pid, G.pid, mg_r16(4 * 4 * n), &bar);
      mg_bulk_g2s(v.S, G.S, mg_r16(8 * 4 * MG_NS * n), &bar);
      mg_bulk_g2s(v.dinv, G.dinv, mg_r16(16 * n), &bar);
    }
    if (A.dense) mg_bulk_g2s(Ainv, A.Ainv, mg_r16(8 * (size_t)nd * nd), &bar);
  }
  __shared__ double om_s[MG_MAXL];
  if (threadIdx.x < MG_MAXL) om_s[threadIdx.x] = __ldcg(&A.ctl->omega[threadIdx.x]);
  // restriction sources of level n_tail (global memory), loaded while the bulk copies fly:
  // pass p, slot q + 4 k of node (threadIdx.x >> 2) + p * MG_TAIL_PASS
  double2 tg[MG_TAIL_P][3];
  {
    const MgLevel& G0 = A.L[l0];
    const int n0 = G0.m.n_nodes;
    const double* tf = A.L[l0 - 1].t;
#pragma unroll
    for (int p = 0; p < MG_TAIL_P; ++p)
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        const int id = (threadIdx.x >> 2) + p * MG_TAIL_PASS, s2 = q + 4 * k;
        const int f = (s2 < 12 && id < n0) ? __ldg(G0.rid + s2 * n0 + id) : -1;
        tg[p][k] = f >= 0 ? GMem::v2(tf, f) : make_double2(0.0, 0.0);
      }
  }
  __syncthreads();
  mg_mbar_wait(&bar, 0);
  TCLK();
  for (int l = l0; l <= c; ++l) {
    const TLevel v = mg_tl(A, l);
    const int n = v.n;
    const double* tf = l == l0 ? nullptr : mg_tl(A, l - 1).t;  // l0 - 1: pre-loaded in tg
    int pass = 0;
    MG_TAIL_NODES(n) {  // b = P^T t_f
      double2 r = make_double2(0.0, 0.0);
      if (id < n) {
#pragma unroll
        for (int k = 0; k < 3; ++k) {
          const int s2 = q + 4 * k;
          if (s2 >= 12) break;
          const int f = v.rid[s2 * n + id];
          if (f < 0) continue;
          double2 t = make_double2(0.0, 0.0);
          if (l == l0) {
#pragma unroll
            for (int p = 0; p < MG_TAIL_P; ++p)
              if (p == pass) t = tg[p][k];
          } else {
            t = ts2(tf, f);
          }
          const double w = mg_rw(s2);
          r.x += w * t.x;
          r.y += w * t.y;
        }
      }
      ++pass;
      r = hw_sum<4>(r);
      if (q == 0 && id < n) d2st(v.b, id, mask2(r, ts2(v.dinv, id)));
    }
    __syncthreads();
    TCLK();
    if (l == c) break;
    const double om = om_s[l];
    MG_TAIL_NODES(n) {  // t = b - A (omega D^-1 b)
      const double2 Av = mg_tapply(v, id, [&](int k) -> double2 {
        const double2 di = ts2(v.dinv, k), bv = ts2(v.b, k);
        return make_double2(om * di.x * bv.x, om * di.y * bv.y);
      });
      if (q == 0 && id < n) {
        const double2 di = ts2(v.dinv, id), bv = ts2(v.b, id);
        d2st(v.t, id, mask2(make_double2(bv.x - Av.x, bv.y - Av.y), di));
      }
    }
    __syncthreads();
    TCLK();
  }
  {  // coarsest solve
    const TLevel v = mg_tl(A, c);
    if (A.dense) {
      for (int i = threadIdx.x; i < nd; i += blockDim.x) {
        double sacc = 0.0;
        for (int j = 0; j < nd; ++j) sacc += Ainv[i * nd + j] * v.b[j];
        v.e[i] = sacc;
      }
      __syncthreads();
    } else {
      const double om = om_s[c];
      double* bufs[2] = {v.e, v.t};
      int cur = (A.nu_c - 1) % 2 == 0 ? 0 : 1;  // the last sweep lands in e
      for (int i = threadIdx.x; i < nd; i += blockDim.x) bufs[cur][i] = om * v.dinv[i] * v.b[i];
      __syncthreads();
      for (int sw = 1; sw < A.nu_c; ++sw) {
        const double* in = bufs[cur];
        double* out = bufs[cur ^ 1];
        MG_TAIL_NODES(v.n) {
          const double2 Ax = mg_tapply(v, id, [&](int k) -> double2 { return ts2(in, k); });
          if (q == 0 && id < v.n) {
            const double2 x = ts2(in, id), di = ts2(v.dinv, id), bv = ts2(v.b, id);
            d2st(out, id, make_double2(x.x + om * di.x * (bv.x - Ax.x), x.y + om * di.y * (bv.y - Ax.y)));
          }
        }
        cur ^= 1;
        __syncthreads();
      }
    }
    TCLK();
    if (l0 == c)  // only the coarsest level in the tail: hand its result to the grid
      for (int i = threadIdx.x; i < nd; i += blockDim.x) A.L[c].e[i] = v.e[i];
  }
  for (int l = c - 1; l >= l0; --l) {
    const TLevel v = mg_tl(A, l), vc = mg_tl(A, l + 1);
    const int n = v.n;
    const double om = om_s[l];
    MG_TAIL_NODES(n) {  // y = omega D^-1 b + P e_c (into t)
      double2 r = make_double2(0.0, 0.0), cnt = make_double2(0.0, 0.0);
      if (id < n) {
        const int k = v.pid[q * n + id];
        if (k >= 0) {
          r = ts2(vc.e, k);
          cnt.x = 1.0;
        }
      }
      r = hw_sum<4>(r);
      cnt = hw_sum<4>(cnt);
      if (q == 0 && id < n) {
        const double w = 1.0 / cnt.x;
        const double2 di = ts2(v.dinv, id), bv = ts2(v.b, id);
        d2st(v.t, id, mask2(make_double2(om * di.x * bv.x + w * r.x, om * di.y * bv.y + w * r.y), di));
      }
    }
    __syncthreads();
    TCLK();
    double* eout = (l == l0) ? A.L[l].e : v.e;
    MG_TAIL_NODES(n) {  // e = y + omega D^-1 (b - A y)
      const double2 Ay = mg_tapply(v, id, [&](int k) -> double2 { return ts2(v.t, k); });
      if (q == 0 && id < n) {
        const double2 y = ts2(v.t, id), di = ts2(v.dinv, id), bv = ts2(v.b, id);
        d2st(eout, id, make_double2(y.x + om * di.x * (bv.x - Ay.x), y.y + om * di.y * (bv.y - Ay.y)));
      }
    }
    __syncthreads();
    TCLK();
  }
}

__global__ void __launch_bounds__(MG_NT, 2) k_mg_fine_smooth(MgArgs A) {
  __shared__ MgWarp ws[MG_WARPS];
  __shared__ double red[MG_WARPS];
  const double om = __ldcg(&A.ctl->omega[0]);
  double rz = 0.0;
  FineSmooth op{{&A.C, A.flags, A.d, A.L[0].dinv, A.phys, A.bq}, om, A.r, A.z, &A.L[0].m, &A.L[1].m,
                A.L[1].e, &rz, {}};
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
  FinePcg op{{&A.C, A.flags, A.d, A.L[0].dinv, A.phys, A.bq}, first ? 0.0 : rho[0] / __ldcg(&A.ctl->rho_prev),
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

// scalar phase-field vectors <-> the two-component layout of the phys-1 instance
__global__ void __launch_bounds__(MG_NT) k_mg_pack2(double* __restrict__ dst2,
                                                    const double* __restrict__ src, long long n) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    reinterpret_cast<double2*>(dst2)[i] = make_double2(src[i], 0.0);
}
__global__ void __launch_bounds__(MG_NT) k_mg_unpack_add(double* __restrict__ x,
                                                         double* __restrict__ target,
                                                         const double* __restrict__ x2,
                                                         long long n) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const double v = __ldg(x2 + 2 * i);
    x[i] = v;
    target[i] += v;
  }
}

// ================================================================================================
// setup kernels: Galerkin cell matrices, inverse diagonals, lambda_max by power steps, dense
// inverse of the coarsest level
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
        if (fe >= 0 && fb != 0.0) {
          const FineBase fop{&A.C, A.flags, A.d, A.L[0].dinv, A.phys, A.bq};
          fop.cell(fe, v, dc, f);
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          col[2 * q] = di[q].x != 0.0 ? f[q].x : 0.0;
          col[2 * q + 1] = di[q].y != 0.0 ? f[q].y : 0.0;
        }
      } else {
        const int fe = mg_cell(mf, ci, cj);
        const double* Kf = A.L[lc - 1].K + 64 * (size_t)fe;
#pragma unroll
        for (int a = 0; a < 8; ++a) col[a] = fe >= 0 ? __ldg(Kf + a * 8 + bcol) : 0.0;
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

// two CTAs per SM (128 registers, 224 B stack): hierarchy setup cfg5 119.9 -> 106.1 ms, cfg3
// 2.33 -> 2.05 ms (one CTA with 167 registers left the per-cell latency chains exposed; three
// CTAs at 80 registers spill 464 B and land in between)
#ifndef PFB_MG_GAL_MINB
#define PFB_MG_GAL_MINB 2
#endif
__global__ void __launch_bounds__(MG_NT, PFB_MG_GAL_MINB) k_mg_galerkin(MgArgs A, int lc) {
  __shared__ MgGal sg[MG_WARPS];
  mg_galerkin(A, lc, blockIdx.x * MG_WARPS + (threadIdx.x >> 5), gridDim.x * MG_WARPS,
              sg[threadIdx.x >> 5]);
}
// power step k (1..MG_POW): blocks [0, fine_blocks) march the fine level, the rest gather the
// coarse levels (concatenated item space)
// three CTAs per SM (80 registers, 296 B stack): setup cfg5 106.1 -> 95.6 ms, cfg3 2.06 -> 1.88 ms
#ifndef PFB_MG_POW_MINB
#define PFB_MG_POW_MINB 3
#endif
__global__ void __launch_bounds__(MG_NT, PFB_MG_POW_MINB) k_mg_pow(MgArgs A, int step, int fine_blocks) {
  __shared__ MgWarp ws[MG_WARPS];
  const int warp = threadIdx.x >> 5;
  auto vin = [&](const MgLevel& L) -> const double* {
    return step == 1 ? nullptr : (((step - 1) & 1) ? L.t : L.e);
  };
  auto vout = [&](const MgLevel& L) -> double* { return (step & 1) ? L.t : L.e; };
  if ((int)blockIdx.x < fine_blocks) {
    FinePow op{{&A.C, A.flags, A.d, A.L[0].dinv, A.phys, A.bq}, vin(A.L[0]), vout(A.L[0])};
    const int w = blockIdx.x * MG_WARPS + warp;
    if (w < A.g0.n_units) mg_march(A.L[0].m, A.g0, w, op, ws[warp]);
    return;
  }
  // coarse levels: concatenated thread space, lpn threads per node on each level (every
  // level starts on a warp boundary, so the lanes of a node share a warp)
  const int t = (blockIdx.x - fine_blocks) * MG_NT + threadIdx.x;
  if (t >= A.coarse_items) return;
  int l = 1;
  while (l + 1 < A.n_levels && t >= A.L[l + 1].item_off) ++l;
  const MgLevel& L = A.L[l];
  const int q = t - L.item_off;
  if (L.lpn == 16) mg_spow<16>(L, vin(L), vout(L), q >> 4);
  else if (L.lpn == 4) mg_spow<4>(L, vin(L), vout(L), q >> 2);
  else mg_spow<1>(L, vin(L), vout(L), q);
}
// omega_l = 4 / (3 lambda_l), lambda_l = ||v_npow|| / ||v_npow-1|| (per-level partials)
__global__ void __launch_bounds__(MG_NT) k_mg_lambda(MgArgs A, int npow) {
  __shared__ double red[MG_WARPS * 2 * MG_MAXL];
  double v[2 * MG_MAXL];
#pragma unroll
  for (int l = 0; l < 2 * MG_MAXL; ++l) v[l] = 0.0;
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long nth = (long long)gridDim.x * blockDim.x;
#pragma unroll
  for (int l = 0; l < MG_MAXL; ++l) {
    if (l >= A.n_levels) break;
    const double* a1 = (npow & 1) ? A.L[l].t : A.L[l].e;
    const double* a0 = (npow & 1) ? A.L[l].e : A.L[l].t;
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
  __shared__ int cn[MG_DENSE_MAX][4];  // corner node ids of the coarsest cells (<= nodes)
  __shared__ int ncell;
  const int c = A.n_levels - 1;
  const DMesh& m = A.L[c].m;
  const int nd = 2 * m.n_nodes;
  if (threadIdx.x == 0) {
    int e = 0;
    for (int cjr = 0; cjr < m.ny; ++cjr) {
      const int4 er = __ldg(m.erow + cjr);
      for (int cir = er.x; cir < er.y && e < MG_DENSE_MAX; ++cir, ++e) {
        cn[e][0] = mg_node(m, cir, cjr, true);
        cn[e][1] = mg_node(m, cir + 1, cjr, true);
        cn[e][2] = mg_node(m, cir + 1, cjr + 1, false);
        cn[e][3] = mg_node(m, cir, cjr + 1, false);
      }
    }
    ncell = e;
  }
  __syncthreads();
  for (int ij = threadIdx.x; ij < nd * nd; ij += blockDim.x) {
    const int i = ij / nd, j = ij % nd;
    const int ni = i >> 1, nj = j >> 1, ci = i & 1, cj = j & 1;
    double s = 0.0;
    for (int e = 0; e < ncell; ++e) {  // cells in id order (row-compact numbering)
      int ka = -1, kb = -1;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        if (cn[e][q] == ni) ka = q;
        if (cn[e][q] == nj) kb = q;
      }
      if (ka >= 0 && kb >= 0)
        s += __ldcg(A.L[c].K + 64 * (size_t)e + (2 * ka + ci) * 8 + 2 * kb + cj);
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
