// pf_mgs.cuh — native scalar geometric-multigrid PCG for the phase-field Newton systems
// (solve_evolution, schemes.py:242-313: K_dd = sum N b N^T w + grad_w sum gradN gradN^T w,
// assembly.py:233-246, masked at the pinned nodes, assembly.py:279-312).
//
// Same system, x0 = 0 and stopping test as the reference's Jacobi-PCG switch
// (linsolve.py:48-54; SciPy 1.18.1 cg: stop at the top of an iteration when the recursive
// residual satisfies ||r|| < rtol ||b||, maxiter 20 n); the preconditioner is one symmetric
// V(1,1)-cycle.  Round 1 ran these solves through the two-component momentum machinery with the
// y dofs dead (pf_mg.cuh, phys 1): every vector, diagonal and restriction was double2 and every
// coarse stencil a 2x2 block, twice the fine-level and four times the coarse-level traffic of the
// scalar field, and 8x8 Galerkin products per coarse cell.  This is the scalar hierarchy:
//   * level 0: the matrix-free phase-field operator (evo_cell_apply: per-Gauss-point Newton
//     coefficient b of k_evo_prepare + the constant gradient block), marched by warps
//     (mg_march of pf_mg.cuh with the value in the x lane);
//   * level l+1: 2x2 agglomeration of level l's cells (L-panel rows and the slit kept, as in
//     pf_mg.cuh), bilinear prolongation masked at pinned / dead nodes, Galerkin cell matrices
//     K_E = sum_c Q_c^T K_c Q_c (4x4 per coarse cell, one thread per coarse cell);
//   * assembled 10-slot scalar stencils (3x3 + the slit tip's second face); grid levels read
//     them in FP32 (preconditioner only: the PCG's operator, residual recurrence, dot products
//     and stopping test stay FP64), the single-CTA tail in FP64 from shared memory;
//   * damped Jacobi V(1,1) with omega_l = 4 / (3 lambda_l), lambda_l from MGS_POW power steps;
//   * coarsest level by a dense inverse (<= MGS_DENSE_MAX nodes) or nu_c Jacobi sweeps.
// Reductions: per-CTA partials summed in a fixed order (bit-reproducible run to run).
#pragma once

namespace pfb {

constexpr int MGS_DENSE_MAX = 64;  // coarsest level by a dense inverse when n_nodes <= this
constexpr int MGS_TAIL_P = 2;      // node passes of the tail's top level (MG_TAIL_NT / 4 each)
// power steps per setup: 4 from a hashed start.  The estimate of lambda_max(D^-1 A) is then a
// little low, omega = 4 / (3 lambda) a little larger -- and the V-cycle better: cfg5 load steps
// 3-6 need 140-143 phase-field iterations with 4 steps, 147-166 with 6, 154-173 with 8 and
// 153-185 with 3 (PFB200_MGS_POW)
constexpr int MGS_POW = 4;

struct MgsLevel {
  DMesh m;
  double* K;      // [n_elems][16] Galerkin cell matrices (l >= 1)
  double* dinv;   // [n] inverse diagonal (0: pinned / dead node)
  double* b;      // right-hand side (l >= 1)
  double* t;      // residual / prolongated iterate / power-iteration buffer
  double* e;      // correction / power-iteration buffer
  const int* nbr; // [MG_NS][n] stencil neighbours (l >= 1)
  double* S;      // [MG_NS][n] FP64 stencil (tail levels)
  float* Sf;      // [MG_NS][n] FP32 stencil (grid levels)
  const int* rid; // [12][n] restriction sources on level l-1
  const int* pid; // [4][n] prolongation sources on level l+1
  double* ev;     // [n] start vector of the power steps when pow_warm (experiments; unused)
  int items, item_off, lpn, in_tail;
};

struct MgsArgs {
  Consts C;
  int n_levels, n_tail, dense, nu_c;
  MgsLevel L[MG_MAXL];
  MarchGeom g0;               // fine-level march units (smoothing, direction, power steps)
  MarchGeom g0r;              // fine-level march units of the residual march
  int coarse_items;
  int pow_warm;               // 1: power steps start from L[l].ev (the previous setup's vectors)
  const double* bq;           // level-0 Newton coefficient per Gauss point [n_elems][4]
  double *x, *r, *z, *p0, *p1, *q;
  double* Ainv;               // [nd*nd] dense inverse of the coarsest level
  double* part;
  MgCtl* ctl;
  const MgIn* in;
  CgResult* result;
  long long n;                // fine nodes
  cudaGraphConditionalHandle cond;
  int use_cond;
  MgTailSlot ts[MG_MAXL];
  int ts_ainv, ts_bytes;
};

__device__ __forceinline__ double mgs_mask(double v, double di) { return di != 0.0 ? v : 0.0; }

// ---- fine level (level 0): scalar node ops for mg_march (value in the x lane, y = 0) --------
struct SFineBase {
  const Consts* C;
  const double* bq;
  const double* dinv;
  struct CRaw {
    double2 b01, b23;
  };
  __device__ void cfetch(int eid, CRaw& c) const {  // one row step ahead (mg_march)
    c.b01 = __ldg(reinterpret_cast<const double2*>(bq) + 2 * eid);
    c.b23 = __ldg(reinterpret_cast<const double2*>(bq) + 2 * eid + 1);
  }
  __device__ void cellr(int, const CRaw& c, const double2 (&v)[4], const double (&)[4],
                        double2 (&f)[4]) const {
    const double pc[4] = {v[0].x, v[1].x, v[2].x, v[3].x};
    const double bb[4] = {c.b01.x, c.b01.y, c.b23.x, c.b23.y};
    double fx[4];
    evo_cell_apply(*C, pc, bb, fx);
#pragma unroll
    for (int k = 0; k < 4; ++k) f[k] = make_double2(fx[k], 0.0);
  }
  __device__ double di(int id) const { return __ldg(dinv + id); }
  // the cells read only the x lane: y and aux carry a node's own data from fetch to out
  static constexpr bool VY = false, AUX = false;
};

struct SFineResid : SFineBase {  // x = omega D^-1 r (pre-smoothing from zero), t = r - A x
  double om;
  const double* r;
  double* t;
  struct Raw {
    double dv, bv;
  };
  __device__ void fetch(int id, int, int, bool, Raw& w) const {
    w.dv = di(id);
    w.bv = __ldg(r + id);
  }
  // the march carries (value, node datum) pairs; the scalar field leaves the y lane free, so
  // it brings each node's own residual (NaN at masked nodes) from fetch to out: no reload there
  __device__ double2 finish(const Raw& w, int, int, int, bool, double& aux) const {
    aux = 0.0;
    return make_double2(om * w.dv * w.bv, w.dv != 0.0 ? w.bv : __longlong_as_double(~0LL));
  }
  __device__ double2 in(int id, int i, int j, bool dup, double& aux) const {
    aux = 0.0;
    if (id < 0) return make_double2(0.0, 0.0);
    Raw w;
    fetch(id, i, j, dup, w);
    return finish(w, id, i, j, dup, aux);
  }
  __device__ void out(int id, double2 Av, double2 v) const {
    t[id] = v.y == v.y ? v.y - Av.x : 0.0;
  }
};

struct SFineSmooth : SFineBase {  // y = omega D^-1 r + P e_1, z = y + omega D^-1 (r - A y); r.z
  double om;
  const double* r;
  double* z;
  const DMesh* mf;
  const DMesh* mc;
  const double* ec;
  double* rz;
  mutable ProlongMarch<double> pm;  // coarse sources of the bilinear prolongation (pf_mg.cuh)
  struct Raw {
    double dv, bv;
  };
  __device__ void fetch(int id, int i, int j, bool, Raw& w) const {
    w.dv = di(id);
    w.bv = __ldg(r + id);
    pm.fetch(*mf, *mc, ec, i, j);
  }
  __device__ double2 smooth0(const Raw& w, double pe) const {
    return make_double2(mgs_mask(om * w.dv * w.bv + pe, w.dv), om * w.dv);  // y, omega D^-1
  }
  // the scalar march's aux value is free: it carries the node's own r from fetch to out
  __device__ double2 finish(const Raw& w, int, int i, int j, bool, double& aux) const {
    aux = w.bv;
    return smooth0(w, pm.value(i, j));
  }
  __device__ double2 in(int id, int i, int j, bool dup, double& aux) const {
    aux = 0.0;
    if (id < 0) return make_double2(0.0, 0.0);
    Raw w;
    w.dv = di(id);
    w.bv = __ldg(r + id);
    aux = w.bv;
    return smooth0(w, ProlongMarch<double>::direct(*mf, *mc, ec, i, j, dup));
  }
  __device__ void outa(int id, double2 Av, double2 y, double bv) const {
    const double ev = y.x + y.y * (bv - Av.x);
    z[id] = ev;
    *rz += bv * ev;
  }
  __device__ void out(int id, double2 Av, double2 y) const { outa(id, Av, y, __ldg(r + id)); }
};

struct SFinePow : SFineBase {  // power step vout = D^-1 A vin (vin == nullptr: hashed start)
  const double* vin;
  double* vout;
  struct Raw {
    double v, dv;
  };
  __device__ void fetch(int id, int, int, bool, Raw& w) const {
    w.v = vin ? __ldg(vin + id) : mg_hash01(2u * id + 1u);
    w.dv = di(id);
  }
  __device__ double2 finish(const Raw& w, int, int, int, bool, double& aux) const {
    aux = 0.0;
    return make_double2(mgs_mask(w.v, w.dv), w.dv);
  }
  __device__ double2 in(int id, int i, int j, bool dup, double& aux) const {
    aux = 0.0;
    if (id < 0) return make_double2(0.0, 0.0);
    Raw w;
    fetch(id, i, j, dup, w);
    return finish(w, id, i, j, dup, aux);
  }
  __device__ void out(int id, double2 Av, double2 v) const { vout[id] = v.y * Av.x; }
};

struct SFinePcg : SFineBase {  // p = z + beta p_old (owner stores), q = A p (masked), p.q
  double beta;
  const double* z;
  const double* pold;
  double* pnew;
  double* q;
  double* pq;
  const DMesh* own = nullptr;  // row strips: p.q over owned nodes only (pf_mgd.cuh)
  struct Raw {
    double zv, po, dv;
  };
  __device__ void fetch(int id, int, int, bool, Raw& w) const {
    w.zv = __ldg(z + id);
    w.po = pold ? __ldg(pold + id) : 0.0;
    w.dv = di(id);
  }
  __device__ double2 finish(const Raw& w, int, int, int, bool, double& aux) const {
    aux = 0.0;
    return make_double2(pold ? w.zv + beta * w.po : w.zv, w.dv);  // p, D^-1 (the mask)
  }
  __device__ double2 in(int id, int i, int j, bool dup, double& aux) const {
    aux = 0.0;
    if (id < 0) return make_double2(0.0, 0.0);
    Raw w;
    fetch(id, i, j, dup, w);
    return finish(w, id, i, j, dup, aux);
  }
  __device__ void out(int id, double2 Av, double2 p) const {
    const double qv = mgs_mask(Av.x, p.y);
    pnew[id] = p.x;
    q[id] = qv;
    if (!own || node_owned(*own, id)) *pq += p.x * qv;
  }
};

// ---- k_evo_prepare as a warp march (big meshes) ---------------------------------------------
// The tile kernel k_evo_prepare (pf_kernels.cuh) stages a node tile with its halo in shared
// memory, passes twice over the tile's cells and runs at ~0.2 of the HBM rate on meshes far
// beyond L2; on those the same quantities come out of one warp march: the value pair is
// (d, d_prev), the cell contributions carry the residual in x and the diagonal in y, each node
// sums them in the reference's element order, the free-node flag rides in the aux value.
// b of a cell in two units' halo is written by both (identical values).
struct EvoPrepOp {
  static constexpr bool VY = true, AUX = false;  // (d, d_prev) per node; aux: the free-node flag
  const Consts* C;
  const double *d, *dprev, *psi, *trp, *dev2, *psimax;
  const uint8_t* pmask;
  double *R, *r, *x, *dinv, *b, *diag;
  int full, extra;
  double *rr, *ngate, *nonpos;
  struct Raw {
    double dv, pv;
    unsigned fr;
  };
  struct CRaw {
    double2 p01, p23;
  };
  __device__ void fetch(int id, int, int, bool, Raw& w) const {
    w.dv = __ldg(d + id);
    w.pv = __ldg(dprev + id);
    w.fr = __ldg(pmask + id);
  }
  __device__ double2 finish(const Raw& w, int, int, int, bool, double& aux) const {
    aux = w.fr ? 1.0 : 0.0;
    return make_double2(w.dv, w.pv);
  }
  __device__ double2 in(int id, int i, int j, bool dup, double& aux) const {
    aux = 0.0;
    if (id < 0) return make_double2(0.0, 0.0);
    Raw w;
    fetch(id, i, j, dup, w);
    return finish(w, id, i, j, dup, aux);
  }
  __device__ void cfetch(int eid, CRaw& c) const {
    c.p01 = __ldg(reinterpret_cast<const double2*>(psi) + 2 * eid);
    c.p23 = __ldg(reinterpret_cast<const double2*>(psi) + 2 * eid + 1);
  }
  // residual (assembly.py:217-228), b (:233-239, schemes.py:112-142), diagonal of K_dd (+ K~)
  __device__ void cellr(int eid, const CRaw& c, const double2 (&v)[4], const double (&)[4],
                        double2 (&f)[4]) const {
    const Consts& K = *C;
    const double dc[4] = {v[0].x, v[1].x, v[2].x, v[3].x};
    const double ps[4] = {c.p01.x, c.p01.y, c.p23.x, c.p23.y};
    double dg[4], pg[4], aw[4];
    interp_q4(K, dc[0], dc[1], dc[2], dc[3], dg);
    interp_q4(K, v[0].y, v[1].y, v[2].y, v[3].y, pg);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const double xq = dg[q] - pg[q];
      const double pen = K.gamma * (0.5 * (xq - fabs(xq)));
      const double src = K.at2 ? (K.src_base * 2.0) * dg[q] : K.src_base;
      aw[q] = (-2.0 * (1.0 - dg[q]) * ps[q] + src + pen) * K.w;
    }
    double res[4], dia[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
    for (int aa = 0; aa < 4; ++aa) {
      double s2 = K.N[0][aa] * aw[0] + K.N[1][aa] * aw[1] + K.N[2][aa] * aw[2] +
                  K.N[3][aa] * aw[3];
      s2 += K.lap[aa][0] * dc[0] + K.lap[aa][1] * dc[1] + K.lap[aa][2] * dc[2] +
            K.lap[aa][3] * dc[3];
      res[aa] = s2;
    }
    if (full) {
      double bq[4], tp[4], dv2[4], pm[4];
      const double srcd = K.at2 ? K.src_base * 2.0 : 0.0;
      if (extra) {
        load4(trp, eid, tp);
        load4(dev2, eid, dv2);
        load4(psimax, eid, pm);
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        bq[q] = 2.0 * ps[q] + srcd + K.gamma * (dg[q] < pg[q] ? 1.0 : 0.0);
        if (extra && gate_gp(K, ps[q], pm[q], dg[q])) {
          bq[q] = bq[q] + extra_gp(K, extra, dg[q], tp[q], dv2[q]);
          *ngate += 1.0;  // only its sign is used (cells in a halo count twice)
        }
      }
      store4(b, eid, bq);
#pragma unroll
      for (int aa = 0; aa < 4; ++aa)
        dia[aa] = K.Nw[0][aa] * K.N[0][aa] * bq[0] + K.Nw[1][aa] * K.N[1][aa] * bq[1] +
                  K.Nw[2][aa] * K.N[2][aa] * bq[2] + K.Nw[3][aa] * K.N[3][aa] * bq[3] +
                  K.lap[aa][aa];
    }
#pragma unroll
    for (int aa = 0; aa < 4; ++aa) f[aa] = make_double2(res[aa], dia[aa]);
  }
  __device__ void outa(int id, double2 Av, double2, double aux) const {
    const bool fr = aux != 0.0;
    const double Rv = Av.x;
    if (R) R[id] = Rv;
    if (fr) *rr += Rv * Rv;
    if (full) {
      r[id] = fr ? -Rv : 0.0;
      x[id] = 0.0;
      if (diag) diag[id] = Av.y;
      if (fr && !(Av.y > 0.0)) *nonpos += 1.0;
      dinv[id] = fr ? 1.0 / Av.y : 0.0;
    }
  }
  __device__ void out(int id, double2 Av, double2 v) const {
    outa(id, Av, v, __ldg(pmask + id) ? 1.0 : 0.0);
  }
};

// partials[3 * block + {0, 1, 2}] = (sum of free R^2, gated Gauss points, free nodes with a
// non-positive diagonal), like k_evo_prepare
__global__ void __launch_bounds__(MG_NT, 2) k_evo_prepare_march(EvoPrepArgs a, MarchGeom g) {
  __shared__ MgWarp ws[MG_WARPS];
  __shared__ double red[MG_WARPS * 3];
  double rr = 0.0, ngate = 0.0, nonpos = 0.0;
  EvoPrepOp op{&a.C, a.d, a.dprev, a.psi, a.trp, a.dev2, a.psimax, a.pmask, a.R, a.r, a.x,
               a.dinv, a.b, a.diag, a.full, a.extra_scheme, &rr, &ngate, &nonpos};
  const int w = blockIdx.x * MG_WARPS + (threadIdx.x >> 5);
  if (w < g.n_units) mg_march(a.m, g, w, op, ws[threadIdx.x >> 5]);
  double v[3] = {rr, ngate, nonpos};
  mg_block_sum<3>(v, red);
  if (threadIdx.x == 0) {
    a.partials[3 * blockIdx.x + 0] = v[0];
    a.partials[3 * blockIdx.x + 1] = v[1];
    a.partials[3 * blockIdx.x + 2] = v[2];
  }
}

// ---- coarse levels: node kernels of the assembled scalar form -------------------------------
template <int W>
__device__ __forceinline__ double hw_sum1(double v) {  // butterfly over W aligned lanes
#pragma unroll
  for (int o = W / 2; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
template <int LPN>
__device__ __forceinline__ double nm_sum1(double v) { return LPN == 1 ? v : hw_sum1<LPN>(v); }

// slot s2 of S x[nbr] at node id (FP32 stencil of the grid levels)
template <class X>
__device__ __forceinline__ double mgs_slot_apply(const MgsLevel& L, int n, int id, int s2,
                                                 X&& xval) {
  if (s2 >= MG_NS || id >= n) return 0.0;
  const int k = __ldg(L.nbr + (size_t)s2 * n + id);
  if (k < 0) return 0.0;
  return (double)__ldg(L.Sf + (size_t)s2 * n + id) * xval(k);
}
template <int LPN, class X>
__device__ __forceinline__ double mgs_apply(const MgsLevel& L, int n, int id, X&& xval) {
  double acc = 0.0;
#pragma unroll
  for (int s2 = NodeMap<LPN>::lane(); s2 < MG_NS; s2 += LPN) acc += mgs_slot_apply(L, n, id, s2, xval);
  return nm_sum1<LPN>(acc);
}

// restriction b = P^T t_{l-1} (masked)
template <int LPN>
__global__ void __launch_bounds__(MG_NT) k_mgs_srestrict(MgsArgs A, int l) {
  const MgsLevel& L = A.L[l];
  const int n = L.m.n_nodes;
  const double* tf = A.L[l - 1].t;
  MG_FOR_NODE_L(n) {
    double v = 0.0;
    if (id < n) {
#pragma unroll
      for (int s2 = NodeMap<LPN>::lane(); s2 < 12; s2 += LPN) {
        const int f = __ldg(L.rid + (size_t)s2 * n + id);
        if (f >= 0) v += mg_rw(s2) * __ldg(tf + f);
      }
    }
    v = nm_sum1<LPN>(v);
    if (MG_LEAD) L.b[id] = mgs_mask(v, __ldg(L.dinv + id));
  }
}
// t = b - A x, x = omega D^-1 b
template <int LPN>
__global__ void __launch_bounds__(MG_NT) k_mgs_sresid(MgsArgs A, int l) {
  const MgsLevel& L = A.L[l];
  const int n = L.m.n_nodes;
  const double om = __ldcg(&A.ctl->omega[l]);
  MG_FOR_NODE_L(n) {
    const double Av = mgs_apply<LPN>(L, n, id, [&](int k) -> double {
      return om * __ldg(L.dinv + k) * __ldg(L.b + k);
    });
    if (MG_LEAD) L.t[id] = mgs_mask(__ldg(L.b + id) - Av, __ldg(L.dinv + id));
  }
}
// y = omega D^-1 b + P e_{l+1} (into t)
template <int LPN>
__global__ void __launch_bounds__(MG_NT) k_mgs_sprolongate(MgsArgs A, int l) {
  const MgsLevel& L = A.L[l];
  const int n = L.m.n_nodes;
  const double om = __ldcg(&A.ctl->omega[l]);
  const double* ec = A.L[l + 1].e;
  MG_FOR_NODE_L(n) {
    double v = 0.0, cnt = 0.0;
    if (id < n) {
#pragma unroll
      for (int s2 = NodeMap<LPN>::lane(); s2 < 4; s2 += LPN) {
        const int c = __ldg(L.pid + (size_t)s2 * n + id);
        if (c >= 0) {
          v += __ldg(ec + c);
          cnt += 1.0;
        }
      }
    }
    v = nm_sum1<LPN>(v);
    cnt = nm_sum1<LPN>(cnt);
    if (MG_LEAD) {
      const double di = __ldg(L.dinv + id);
      L.t[id] = mgs_mask(om * di * __ldg(L.b + id) + v / cnt, di);
    }
  }
}
// e = y + omega D^-1 (b - A y), y in t
template <int LPN>
__global__ void __launch_bounds__(MG_NT) k_mgs_ssmooth(MgsArgs A, int l) {
  const MgsLevel& L = A.L[l];
  const int n = L.m.n_nodes;
  const double om = __ldcg(&A.ctl->omega[l]);
  MG_FOR_NODE_L(n) {
    const double Ay = mgs_apply<LPN>(L, n, id, [&](int k) -> double { return __ldg(L.t + k); });
    if (MG_LEAD)
      L.e[id] = __ldg(L.t + id) + om * __ldg(L.dinv + id) * (__ldg(L.b + id) - Ay);
  }
}
// fused down-sweep of a small level: the restriction of t_{l-1} evaluated at each neighbour by
// the lane that multiplies it, x = omega D^-1 b, t = b - A x; b stored for the up-sweep
template <int LPN>
__global__ void __launch_bounds__(MG_NT) k_mgs_sdown(MgsArgs A, int l) {
  const MgsLevel& L = A.L[l];
  const int n = L.m.n_nodes;
  const double om = __ldcg(&A.ctl->omega[l]);
  const double* tf = A.L[l - 1].t;
  MG_FOR_NODE_L(n) {
    double acc = 0.0, bc = 0.0;
    if (id < n) {
#pragma unroll
      for (int s2 = NodeMap<LPN>::lane(); s2 < MG_NS; s2 += LPN) {
        const int k = __ldg(L.nbr + (size_t)s2 * n + id);
        if (k < 0) continue;
        int f[12];
#pragma unroll
        for (int j = 0; j < 12; ++j) f[j] = __ldg(L.rid + (size_t)j * n + k);
        double b = 0.0;
#pragma unroll
        for (int j = 0; j < 12; ++j)
          if (f[j] >= 0) b += mg_rw(j) * __ldg(tf + f[j]);
        const double di = __ldg(L.dinv + k);
        b = mgs_mask(b, di);
        if (s2 == 4) bc = b;
        acc += (double)__ldg(L.Sf + (size_t)s2 * n + id) * (om * di * b);
      }
    }
    acc = nm_sum1<LPN>(acc);
    bc = nm_sum1<LPN>(bc);
    if (MG_LEAD) {
      L.b[id] = bc;
      L.t[id] = mgs_mask(bc - acc, __ldg(L.dinv + id));
    }
  }
}
// fused up-sweep of a small level: y = omega D^-1 b + P e_{l+1} at each neighbour by its lane,
// e = y + omega D^-1 (b - A y)
template <int LPN>
__global__ void __launch_bounds__(MG_NT) k_mgs_sup(MgsArgs A, int l) {
  const MgsLevel& L = A.L[l];
  const int n = L.m.n_nodes;
  const double om = __ldcg(&A.ctl->omega[l]);
  const double* ec = A.L[l + 1].e;
  MG_FOR_NODE_L(n) {
    double acc = 0.0, yc = 0.0;
    if (id < n) {
#pragma unroll
      for (int s2 = NodeMap<LPN>::lane(); s2 < MG_NS; s2 += LPN) {
        const int k = __ldg(L.nbr + (size_t)s2 * n + id);
        if (k < 0) continue;
        int c[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) c[j] = __ldg(L.pid + (size_t)j * n + k);
        const double w = 1.0 / ((c[0] >= 0) + (c[1] >= 0) + (c[2] >= 0) + (c[3] >= 0));
        double pe = 0.0;
#pragma unroll
        for (int j = 0; j < 4; ++j)
          if (c[j] >= 0) pe += __ldg(ec + c[j]);
        const double di = __ldg(L.dinv + k);
        const double y = mgs_mask(om * di * __ldg(L.b + k) + w * pe, di);
        if (s2 == 4) yc = y;
        acc += (double)__ldg(L.Sf + (size_t)s2 * n + id) * y;
      }
    }
    acc = nm_sum1<LPN>(acc);
    yc = nm_sum1<LPN>(yc);
    if (MG_LEAD) L.e[id] = yc + om * __ldg(L.dinv + id) * (__ldg(L.b + id) - acc);
  }
}
// Jacobi sweep out = in + omega D^-1 (b - A in) (grid coarsest level)
template <int LPN>
__global__ void __launch_bounds__(MG_NT) k_mgs_ssweep(MgsArgs A, int l, const double* in,
                                                      double* out) {
  const MgsLevel& L = A.L[l];
  const int n = L.m.n_nodes;
  const double om = __ldcg(&A.ctl->omega[l]);
  MG_FOR_NODE_L(n) {
    const double Ax = mgs_apply<LPN>(L, n, id, [&](int k) -> double { return __ldg(in + k); });
    if (MG_LEAD) out[id] = __ldg(in + id) + om * __ldg(L.dinv + id) * (__ldg(L.b + id) - Ax);
  }
}
__global__ void __launch_bounds__(MG_NT) k_mgs_jacobi0(MgsArgs A, int l, double* out) {
  const MgsLevel& L = A.L[l];
  const double om = __ldcg(&A.ctl->omega[l]);
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < L.m.n_nodes;
       i += (long long)gridDim.x * blockDim.x)
    out[i] = om * __ldcg(L.dinv + i) * __ldcg(L.b + i);
}
__global__ void __launch_bounds__(MG_NT) k_mgs_coarse_dense(MgsArgs A) {
  const MgsLevel& L = A.L[A.n_levels - 1];
  const int nd = L.m.n_nodes;
  for (int i = threadIdx.x; i < nd; i += blockDim.x) {
    double s = 0.0;
    for (int j = 0; j < nd; ++j) s += __ldcg(A.Ainv + (size_t)i * nd + j) * __ldcg(L.b + j);
    L.e[i] = s;
  }
}

// ---- large coarse levels (>= 2^20 nodes: on smaller, L2-resident levels the table kernels are
// faster, cfg2's 66 k-node level 1 125 vs 112 us per V-cycle), one thread per node over (row,
// 32-column chunk) items: the
// neighbour and restriction ids follow from the row tables where the stencil is
// regular (interior rows of equal extent away from the slit, interior columns); only boundary
// and slit nodes read the index tables.  Same products in the same order as the table kernels
// (bitwise-identical results), about 40 B per node less traffic per stencil product (the
// neighbour ids) and 48 B per restriction.  The prolongation keeps its 16-byte table.
__device__ __forceinline__ bool mgs_regular(const DMesh& m, int i, int j, int4 rw) {
  if (j <= 0 || j >= m.ny || i <= rw.x || i >= rw.y - 1) return false;
  if (m.notch_row >= 0 && j >= m.notch_row - 1 && j <= m.notch_row + 1) return false;
  const int4 a = __ldg(m.nrow + j - 1), b = __ldg(m.nrow + j + 1);
  return a.x == rw.x && a.y == rw.y && b.x == rw.x && b.y == rw.y;
}
template <class X>
__device__ __forceinline__ double mgs_row_apply(const MgsLevel& L, int n, int id, int i, int j,
                                                bool dup, X&& xval) {
  double acc = 0.0;
  const int4 rw = __ldg(L.m.nrow + j);
  if (!dup && mgs_regular(L.m, i, j, rw)) {
    const int len = rw.y - rw.x;
#pragma unroll
    for (int s2 = 0; s2 < 9; ++s2) {
      const int k = id + (s2 / 3 - 1) * len + (s2 % 3 - 1);
      acc += (double)__ldg(L.Sf + (size_t)s2 * n + id) * xval(k);
    }
  } else {
#pragma unroll
    for (int s2 = 0; s2 < MG_NS; ++s2) acc += mgs_slot_apply(L, n, id, s2, xval);
  }
  return acc;
}
#define MGS_GW (int)(blockIdx.x * MG_WARPS + (threadIdx.x >> 5)), (int)(gridDim.x * MG_WARPS)
__global__ void __launch_bounds__(MG_NT) k_mgs_rrestrict(MgsArgs A, int l) {
  const MgsLevel& L = A.L[l];
  const DMesh& mf = A.L[l - 1].m;
  const int n = L.m.n_nodes;
  const double* tf = A.L[l - 1].t;
  mg_for_nodes<GMem>(L.m, MGS_GW, [&](int id, int I, int J, bool dup) {
    double v = 0.0;
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
        const int f = st[s2 / 3] + (i0 + (s2 % 3 - 1) - r0.x);
        v += mg_rw(s2) * __ldg(tf + f);
      }
    } else {
#pragma unroll
      for (int s2 = 0; s2 < 12; ++s2) {
        const int f = __ldg(L.rid + (size_t)s2 * n + id);
        if (f >= 0) v += mg_rw(s2) * __ldg(tf + f);
      }
    }
    L.b[id] = mgs_mask(v, __ldg(L.dinv + id));
  });
}
__global__ void __launch_bounds__(MG_NT) k_mgs_rresid(MgsArgs A, int l) {
  const MgsLevel& L = A.L[l];
  const int n = L.m.n_nodes;
  const double om = __ldcg(&A.ctl->omega[l]);
  mg_for_nodes<GMem>(L.m, MGS_GW, [&](int id, int i, int j, bool dup) {
    const double Av = mgs_row_apply(L, n, id, i, j, dup, [&](int k) -> double {
      return om * __ldg(L.dinv + k) * __ldg(L.b + k);
    });
    L.t[id] = mgs_mask(__ldg(L.b + id) - Av, __ldg(L.dinv + id));
  });
}
__global__ void __launch_bounds__(MG_NT) k_mgs_rsmooth(MgsArgs A, int l) {
  const MgsLevel& L = A.L[l];
  const int n = L.m.n_nodes;
  const double om = __ldcg(&A.ctl->omega[l]);
  mg_for_nodes<GMem>(L.m, MGS_GW, [&](int id, int i, int j, bool dup) {
    const double Ay = mgs_row_apply(L, n, id, i, j, dup, [&](int k) -> double { return __ldg(L.t + k); });
    L.e[id] = __ldg(L.t + id) + om * __ldg(L.dinv + id) * (__ldg(L.b + id) - Ay);
  });
}

// power step of a large one-thread-per-node level with the row-table stencil ids (same sums as
// mgs_spow<1>)
__global__ void __launch_bounds__(MG_NT) k_mgs_rpow(MgsArgs A, int l, int step) {
  const MgsLevel& L = A.L[l];
  const int n = L.m.n_nodes;
  const double* vin = step == 1 ? (A.pow_warm ? L.ev : nullptr) : (((step - 1) & 1) ? L.t : L.e);
  double* vout = (step & 1) ? L.t : L.e;
  mg_for_nodes<GMem>(L.m, MGS_GW, [&](int id, int i, int j, bool dup) {
    const double Av = mgs_row_apply(L, n, id, i, j, dup, [&](int k) -> double {
      const double x = vin ? __ldg(vin + k) : mg_hash01(2u * k + 1u);
      return mgs_mask(x, __ldg(L.dinv + k));
    });
    vout[id] = __ldg(L.dinv + id) * Av;
  });
}

// power step at one node of a coarse level: vout = D^-1 A vin (vin == nullptr: hashed start)
template <int LPN>
__device__ __forceinline__ void mgs_spow(const MgsLevel& L, const double* vin, double* vout,
                                         int id) {
  const int n = L.m.n_nodes;
  double acc = 0.0;
#pragma unroll
  for (int s2 = NodeMap<LPN>::lane(); s2 < MG_NS; s2 += LPN)
    acc += mgs_slot_apply(L, n, id, s2, [&](int k) -> double {
      const double x = vin ? __ldg(vin + k) : mg_hash01(2u * k + 1u);
      return mgs_mask(x, __ldg(L.dinv + k));
    });
  const double Av = nm_sum1<LPN>(acc);
  if (NodeMap<LPN>::lane() == 0 && id < n) vout[id] = __ldg(L.dinv + id) * Av;
}

// ---- setup ----------------------------------------------------------------------------------
// Galerkin cell matrices of level lc from level lc-1, one thread per coarse cell:
// K_E = sum_c Q_c^T K_c Q_c with K_c the child's 4x4 matrix (lc == 1: the fine phase-field cell
// matrix sum_g b_g N_g N_g^T w + the gradient block, rows / columns of masked corners zeroed).
__global__ void __launch_bounds__(MG_NT) k_mgs_galerkin(MgsArgs A, int lc) {
  const DMesh& mc = A.L[lc].m;
  const DMesh& mf = A.L[lc - 1].m;
  const int total = mc.nx * mc.ny;
  for (int it = blockIdx.x * blockDim.x + threadIdx.x; it < total; it += gridDim.x * blockDim.x) {
    const int J = it / mc.nx, I = it % mc.nx;
    const int4 er = __ldg(mc.erow + J);
    if (I < er.x || I >= er.y) continue;
    const int E = er.z + (I - er.x);
    double KE[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) KE[k] = 0.0;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int ci = 2 * I + (c & 1), cj = 2 * J + (c >> 1);
      const int fe = mg_cell(mf, ci, cj);
      if (fe < 0) continue;
      double Kc[16];
      if (lc == 1) {
        int nd[4];
        nd[0] = mg_node(mf, ci, cj, true);
        nd[1] = mg_node(mf, ci + 1, cj, true);
        nd[2] = mg_node(mf, ci + 1, cj + 1, false);
        nd[3] = mg_node(mf, ci, cj + 1, false);
        bool live[4];
#pragma unroll
        for (int a = 0; a < 4; ++a) live[a] = nd[a] >= 0 && __ldg(A.L[0].dinv + nd[a]) != 0.0;
        const double2 b01 = __ldg(reinterpret_cast<const double2*>(A.bq) + 2 * fe);
        const double2 b23 = __ldg(reinterpret_cast<const double2*>(A.bq) + 2 * fe + 1);
        const double bb[4] = {b01.x, b01.y, b23.x, b23.y};
        // the columns of evo_cell_apply (same products, same order)
#pragma unroll
        for (int bcol = 0; bcol < 4; ++bcol) {
          double pc[4] = {0.0, 0.0, 0.0, 0.0};
          pc[bcol] = 1.0;
          double f[4];
          evo_cell_apply(A.C, pc, bb, f);
#pragma unroll
          for (int a = 0; a < 4; ++a) Kc[a * 4 + bcol] = (live[a] && live[bcol]) ? f[a] : 0.0;
        }
      } else {
        const double2* Kf = reinterpret_cast<const double2*>(A.L[lc - 1].K + 16 * (size_t)fe);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const double2 v = __ldg(Kf + k);
          Kc[2 * k] = v.x;
          Kc[2 * k + 1] = v.y;
        }
      }
      // T = K_c Q_c, KE += Q_c^T T
#pragma unroll
      for (int a = 0; a < 4; ++a) {
        double T[4];
#pragma unroll
        for (int B = 0; B < 4; ++B) {
          double s = 0.0;
#pragma unroll
          for (int k2 = 0; k2 < 4; ++k2) s += Kc[a * 4 + k2] * mg_q(c, k2, B);
          T[B] = s;
        }
#pragma unroll
        for (int Ar = 0; Ar < 4; ++Ar) {
          const double qa = mg_q(c, a, Ar);
#pragma unroll
          for (int B = 0; B < 4; ++B) KE[Ar * 4 + B] += qa * T[B];
        }
      }
    }
    double2* out = reinterpret_cast<double2*>(A.L[lc].K + 16 * (size_t)E);
#pragma unroll
    for (int k = 0; k < 8; ++k) out[k] = make_double2(KE[2 * k], KE[2 * k + 1]);
  }
}

// assemble the stencil of level l from its cell matrices (FP32 for grid levels, FP64 for the
// tail), and its inverse diagonal; one thread per node
__global__ void __launch_bounds__(MG_NT) k_mgs_stencil(MgsArgs A, int l) {
  const MgsLevel& L = A.L[l];
  const DMesh& m = L.m;
  const int n = m.n_nodes;
  mg_for_nodes<GMem>(m, blockIdx.x * MG_WARPS + (threadIdx.x >> 5), gridDim.x * MG_WARPS,
                     [&](int id, int i, int j, bool) {
    int nb[MG_NS];
#pragma unroll
    for (int s2 = 0; s2 < MG_NS; ++s2) nb[s2] = __ldg(L.nbr + (size_t)s2 * n + id);
    double acc[MG_NS];
#pragma unroll
    for (int s2 = 0; s2 < MG_NS; ++s2) acc[s2] = 0.0;
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
      const double* Ke = L.K + 16 * (size_t)e;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int qx = ci + ((q == 1 || q == 2) ? 1 : 0) - i, qy = cj + (q >= 2 ? 1 : 0) - j;
        int slot = qy < 0 ? 1 + qx : (qy > 0 ? 7 + qx : 4 + qx);
        if (qy == 0 && nb[slot] != cn[q]) slot = 9;
        const double kv = __ldg(Ke + k * 4 + q);
#pragma unroll
        for (int s2 = 0; s2 < MG_NS; ++s2)
          if (s2 == slot) acc[s2] += kv;
      }
    }
    if (L.in_tail) {
#pragma unroll
      for (int s2 = 0; s2 < MG_NS; ++s2) L.S[(size_t)s2 * n + id] = acc[s2];
    } else {
#pragma unroll
      for (int s2 = 0; s2 < MG_NS; ++s2) L.Sf[(size_t)s2 * n + id] = (float)acc[s2];
    }
    L.dinv[id] = acc[4] > 0.0 ? 1.0 / acc[4] : 0.0;
  });
}

// power step k (1..MG_POW): blocks [0, fine_blocks) march the fine level, the rest gather the
// coarse grid levels (concatenated item space; the tail levels use their FP64 stencils below)
__global__ void __launch_bounds__(MG_NT, 3) k_mgs_pow(MgsArgs A, int step, int fine_blocks) {
  __shared__ MgWarp ws[MG_WARPS];
  const int warp = threadIdx.x >> 5;
  auto vin = [&](const MgsLevel& L) -> const double* {
    return step == 1 ? (A.pow_warm ? L.ev : nullptr) : (((step - 1) & 1) ? L.t : L.e);
  };
  auto vout = [&](const MgsLevel& L) -> double* { return (step & 1) ? L.t : L.e; };
  if ((int)blockIdx.x < fine_blocks) {
    SFinePow op{{&A.C, A.bq, A.L[0].dinv}, vin(A.L[0]), vout(A.L[0])};
    const int w = blockIdx.x * MG_WARPS + warp;
    if (w < A.g0.n_units) mg_march(A.L[0].m, A.g0, w, op, ws[warp]);
    return;
  }
  const int t = (blockIdx.x - fine_blocks) * MG_NT + threadIdx.x;
  if (t >= A.coarse_items) return;
  int l = 1;
  while (l + 1 < A.n_tail && t >= A.L[l + 1].item_off) ++l;
  const MgsLevel& L = A.L[l];
  const int q = t - L.item_off;
  if (L.lpn == 16) mgs_spow<16>(L, vin(L), vout(L), q >> 4);
  else if (L.lpn == 4) mgs_spow<4>(L, vin(L), vout(L), q >> 2);
  else mgs_spow<1>(L, vin(L), vout(L), q);
}
// the coarse grid levels' power step on its own (a light kernel at full occupancy: inside the
// march kernel's register budget it took 2.0 ms per step at cfg5)
// (levels by the row-table kernel k_mgs_rpow come first in the item space: skipped by off0)
__global__ void __launch_bounds__(MG_NT) k_mgs_pow_coarse(MgsArgs A, int step, int off0) {
  const int t = off0 + blockIdx.x * MG_NT + threadIdx.x;
  if (t >= A.coarse_items) return;
  int l = 1;
  while (l + 1 < A.n_tail && t >= A.L[l + 1].item_off) ++l;
  const MgsLevel& L = A.L[l];
  const double* vin = step == 1 ? (A.pow_warm ? L.ev : nullptr) : (((step - 1) & 1) ? L.t : L.e);
  double* vout = (step & 1) ? L.t : L.e;
  const int q = t - L.item_off;
  if (L.lpn == 16) mgs_spow<16>(L, vin, vout, q >> 4);
  else if (L.lpn == 4) mgs_spow<4>(L, vin, vout, q >> 2);
  else mgs_spow<1>(L, vin, vout, q);
}
// power steps of the tail levels (FP64 stencils), one CTA, all MG_POW steps
__global__ void __launch_bounds__(MG_TAIL_NT) k_mgs_pow_tail(MgsArgs A, int npow) {
  for (int step = 1; step <= npow; ++step) {
    for (int l = A.n_tail; l < A.n_levels; ++l) {
      const MgsLevel& L = A.L[l];
      const int n = L.m.n_nodes;
      const double* vin = step == 1 ? (A.pow_warm ? L.ev : nullptr)
                                    : (((step - 1) & 1) ? L.t : L.e);
      double* vout = (step & 1) ? L.t : L.e;
      for (int id = threadIdx.x; id < n; id += blockDim.x) {
        double acc = 0.0;
        for (int s2 = 0; s2 < MG_NS; ++s2) {
          const int k = L.nbr[(size_t)s2 * n + id];
          if (k < 0) continue;
          const double x = vin ? __ldcg(vin + k) : mg_hash01(2u * k + 1u);
          acc += __ldcg(L.S + (size_t)s2 * n + id) * mgs_mask(x, __ldcg(L.dinv + k));
        }
        vout[id] = __ldcg(L.dinv + id) * acc;
      }
    }
    __syncthreads();
  }
}
// omega_l = 4 / (3 lambda_l), lambda_l = ||v_npow|| / ||v_npow-1|| (per-level partials)
__global__ void __launch_bounds__(MG_NT) k_mgs_lambda(MgsArgs A, int npow) {
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
    const long long n = A.L[l].m.n_nodes;
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
// dense inverse of the coarsest level (one CTA): assembled from its cell matrices, Gauss-Jordan
// without pivoting (SPD on the live nodes; dead nodes get identity rows, zeroed afterwards)
__global__ void __launch_bounds__(MG_NT) k_mgs_dense(MgsArgs A) {
  __shared__ double M[MGS_DENSE_MAX * MGS_DENSE_MAX];
  __shared__ double F[MGS_DENSE_MAX];
  __shared__ int live[MGS_DENSE_MAX];
  __shared__ int cn[MGS_DENSE_MAX][4];
  __shared__ int ncell;
  const int c = A.n_levels - 1;
  const DMesh& m = A.L[c].m;
  const int nd = m.n_nodes;
  if (threadIdx.x == 0) {
    int e = 0;
    for (int cjr = 0; cjr < m.ny; ++cjr) {
      const int4 er = __ldg(m.erow + cjr);
      for (int cir = er.x; cir < er.y && e < MGS_DENSE_MAX; ++cir, ++e) {
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
    double s = 0.0;
    for (int e = 0; e < ncell; ++e) {
      int ka = -1, kb = -1;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        if (cn[e][q] == i) ka = q;
        if (cn[e][q] == j) kb = q;
      }
      if (ka >= 0 && kb >= 0) s += __ldcg(A.L[c].K + 16 * (size_t)e + ka * 4 + kb);
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
    for (int j = threadIdx.x; j < nd; j += blockDim.x) M[k * nd + j] = (j == k ? 1.0 : M[k * nd + j]) / piv;
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

// ---- solve ------------------------------------------------------------------------------------
// x0 = 0, r0 = b; ||b|| (scipy: rtol * ||b||); the last CTA sets the control block and the WHILE
// condition
__global__ void __launch_bounds__(MG_NT) k_mgs_init(MgsArgs A) {
  __shared__ double red[MG_WARPS];
  const MgIn* in = A.in;
  double rr = 0.0;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < A.n;
       i += (long long)gridDim.x * blockDim.x) {
    const double rv = __ldcg(A.r + i);
    A.x[i] = 0.0;
    rr += rv * rv;
  }
  double v[1] = {rr};
  if (mg_publish<1>(v, A.part, &A.ctl->count, red)) {
    double tot[1];
    mg_all_reduce<1>(A.part, gridDim.x, red, tot);
    if (threadIdx.x == 0) {
      MgCtl& c = *A.ctl;
      c.count = 0;
      c.rr = tot[0];
      c.maxiter = in->maxiter;
      c.target = in->target;
      c.bnorm = sqrt(tot[0]);
      c.atol = in->rtol * c.bnorm;
      c.k = 0;
      c.rho_prev = 0.0;
      c.status = CG_CONVERGED;
      c.done = (c.bnorm == 0.0 || sqrt(tot[0]) < c.atol) ? 1 : 0;
      if (!c.done && c.maxiter <= 0) { c.done = 1; c.status = CG_MAXITER; }
      if (A.use_cond) cudaGraphSetConditional(A.cond, c.done ? 0u : 1u);
    }
  }
}

#ifndef PFB_MGS_MINB
#define PFB_MGS_MINB 3
#endif
// the residual march is the lightest: four CTAs per SM (its own unit geometry g0r; measured at
// cfg5 0.77 -> 0.66 ms, while the smoothing and direction marches lose at four)
#ifndef PFB_MGS_MINB_RESID
#define PFB_MGS_MINB_RESID 4
#endif
__global__ void __launch_bounds__(MG_NT, PFB_MGS_MINB_RESID) k_mgs_fine_resid(MgsArgs A) {
  __shared__ MgWarp ws[MG_WARPS];
  const double om = __ldcg(&A.ctl->omega[0]);
  SFineResid op{{&A.C, A.bq, A.L[0].dinv}, om, A.r, A.L[0].t};
  const int w = blockIdx.x * MG_WARPS + (threadIdx.x >> 5);
  if (w < A.g0r.n_units) mg_march(A.L[0].m, A.g0r, w, op, ws[threadIdx.x >> 5]);
}

__global__ void __launch_bounds__(MG_NT, PFB_MGS_MINB) k_mgs_fine_smooth(MgsArgs A) {
  __shared__ MgWarp ws[MG_WARPS];
  __shared__ double red[MG_WARPS];
  const double om = __ldcg(&A.ctl->omega[0]);
  double rz = 0.0;
  SFineSmooth op{{&A.C, A.bq, A.L[0].dinv}, om, A.r, A.z, &A.L[0].m, &A.L[1].m, A.L[1].e, &rz, {}};
  const int w = blockIdx.x * MG_WARPS + (threadIdx.x >> 5);
  if (w < A.g0.n_units) mg_march(A.L[0].m, A.g0, w, op, ws[threadIdx.x >> 5]);
  double v[1] = {rz};
  mg_block_sum<1>(v, red);
  if (threadIdx.x == 0) A.part[blockIdx.x] = v[0];  // r.z partials, reduced by k_mgs_pcg
}

#ifndef PFB_MGS_MINB_PCG
#define PFB_MGS_MINB_PCG PFB_MGS_MINB
#endif
__global__ void __launch_bounds__(MG_NT, PFB_MGS_MINB_PCG) k_mgs_pcg(MgsArgs A, int n_rz) {
  __shared__ MgWarp ws[MG_WARPS];
  __shared__ double red[MG_WARPS];
  double rho[1];
  mg_all_reduce<1>(A.part, n_rz, red, rho);
  const long long k = __ldcg(&A.ctl->k);
  const bool first = k == 0;
  double pq = 0.0;
  SFinePcg op{{&A.C, A.bq, A.L[0].dinv}, first ? 0.0 : rho[0] / __ldcg(&A.ctl->rho_prev), A.z,
              first ? nullptr : ((k & 1) ? A.p0 : A.p1), (k & 1) ? A.p1 : A.p0, A.q, &pq};
  const int w = blockIdx.x * MG_WARPS + (threadIdx.x >> 5);
  if (w < A.g0.n_units) mg_march(A.L[0].m, A.g0, w, op, ws[threadIdx.x >> 5]);
  double v[1] = {pq};
  mg_block_sum<1>(v, red);
  if (threadIdx.x == 0) A.part[n_rz + blockIdx.x] = v[0];
}

__global__ void __launch_bounds__(MG_NT) k_mgs_update(MgsArgs A, int n_rz, int n_pq) {
  __shared__ double red[MG_WARPS];
  double rho[1], pq[1];
  mg_all_reduce<1>(A.part, n_rz, red, rho);
  mg_all_reduce<1>(A.part + n_rz, n_pq, red, pq);
  const long long k = __ldcg(&A.ctl->k);
  const double alpha = rho[0] / pq[0];
  const double* p = (k & 1) ? A.p1 : A.p0;
  double rr = 0.0;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < A.n;
       i += (long long)gridDim.x * blockDim.x) {
    const double pv = __ldcg(p + i), qv = __ldcg(A.q + i);
    const double xv = __ldcg(A.x + i) + alpha * pv;
    const double rv = __ldcg(A.r + i) - alpha * qv;
    A.x[i] = xv;
    A.r[i] = rv;
    rr += rv * rv;
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
      // the SPD probe of the gated solves (check_spd, linsolve.py:58-77; pf_cg.cuh k_cg): a
      // direction of non-positive curvature proves that K_dd + K~ is not positive definite,
      // whatever the preconditioner
      if (__ldcg(&A.in->probe) && !(pq[0] > 0.0)) { c.done = 1; c.status = CG_INDEFINITE; }
      else if (rn < c.atol) { c.done = 1; c.status = CG_CONVERGED; }
      else if (!(rn == rn)) { c.done = 1; c.status = CG_NAN; }
      else if (c.k >= c.maxiter) { c.done = 1; c.status = CG_MAXITER; }
      if (A.use_cond) cudaGraphSetConditional(A.cond, c.done ? 0u : 1u);
    }
  }
}

__global__ void __launch_bounds__(MG_NT) k_mgs_finish(MgsArgs A) {
  const MgCtl& c = *A.ctl;
  const int status = __ldcg(&c.status);
  double* target = *(double* volatile*)&c.target;
  if (target && status == CG_CONVERGED)
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < A.n;
         i += (long long)gridDim.x * blockDim.x)
      target[i] += __ldcg(A.x + i);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    A.result->iters = __ldcg(&c.k);
    A.result->status = status;
    A.result->bnorm = __ldcg(&c.bnorm);
    A.result->rnorm = sqrt(__ldcg(&c.rr));
  }
}

// ---- tail: levels [n_tail, n_levels) in shared memory, cycled by one CTA ---------------------
struct STLevel {
  int n;
  const int *nbr, *rid, *pid;
  const double *S, *dinv;
  double *b, *t, *e;
};
__device__ __forceinline__ STLevel mgs_tl(const MgsArgs& A, int l) {
  unsigned char* sm = mg_tail_smem;
  const MgTailSlot& o = A.ts[l];
  STLevel v;
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
template <class X>
__device__ __forceinline__ double mgs_tapply(const STLevel& L, int id, X&& xval) {
  const int q = threadIdx.x & 3, n = L.n;
  double v = 0.0;
  if (id < n) {
#pragma unroll
    for (int s2 = q; s2 < MG_NS; s2 += 4) {
      const int k = L.nbr[s2 * n + id];
      if (k >= 0) v += L.S[s2 * n + id] * xval(k);
    }
  }
  return hw_sum1<4>(v);
}

__global__ void __launch_bounds__(MG_TAIL_NT) k_mgs_tail(MgsArgs A) {
  const int nl = A.n_levels, l0 = A.n_tail, c = nl - 1;
  const int q = threadIdx.x & 3;
  const int nd = A.L[c].m.n_nodes;
  double* Ainv = reinterpret_cast<double*>(mg_tail_smem + A.ts_ainv);
  __shared__ __align__(8) unsigned long long bar;
  if (threadIdx.x == 0) {
    unsigned total = 0;
    for (int l = l0; l < nl; ++l) {
      const size_t n = A.L[l].m.n_nodes;
      total += mg_r16(4 * MG_NS * n) + mg_r16(4 * 12 * n) + (l < c ? mg_r16(4 * 4 * n) : 0) +
               mg_r16(8 * MG_NS * n) + mg_r16(8 * n);
    }
    if (A.dense) total += mg_r16(8 * (size_t)nd * nd);
    mg_mbar_init_expect(&bar, total);
    for (int l = l0; l < nl; ++l) {
      const STLevel v = mgs_tl(A, l);
      const MgsLevel& G = A.L[l];
      const size_t n = v.n;
      mg_bulk_g2s(v.nbr, G.nbr, mg_r16(4 * MG_NS * n), &bar);
      mg_bulk_g2s(v.rid, G.rid, mg_r16(4 * 12 * n), &bar);
      if (l < c) mg_bulk_g2s(v.pid, G.pid, mg_r16(4 * 4 * n), &bar);
      mg_bulk_g2s(v.S, G.S, mg_r16(8 * MG_NS * n), &bar);
      mg_bulk_g2s(v.dinv, G.dinv, mg_r16(8 * n), &bar);
    }
    if (A.dense) mg_bulk_g2s(Ainv, A.Ainv, mg_r16(8 * (size_t)nd * nd), &bar);
  }
  __shared__ double om_s[MG_MAXL];
  if (threadIdx.x < MG_MAXL) om_s[threadIdx.x] = __ldcg(&A.ctl->omega[threadIdx.x]);
  // restriction sources of level n_tail (global memory), loaded while the bulk copies fly
  double tg[MGS_TAIL_P][3];
  {
    const MgsLevel& G0 = A.L[l0];
    const int n0 = G0.m.n_nodes;
    const double* tf = A.L[l0 - 1].t;
#pragma unroll
    for (int p = 0; p < MGS_TAIL_P; ++p)
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        const int id = (threadIdx.x >> 2) + p * MG_TAIL_PASS, s2 = q + 4 * k;
        const int f = (s2 < 12 && id < n0) ? __ldg(G0.rid + s2 * n0 + id) : -1;
        tg[p][k] = f >= 0 ? __ldcg(tf + f) : 0.0;
      }
  }
  __syncthreads();
  mg_mbar_wait(&bar, 0);
  for (int l = l0; l <= c; ++l) {
    const STLevel v = mgs_tl(A, l);
    const int n = v.n;
    const double* tf = l == l0 ? nullptr : mgs_tl(A, l - 1).t;
    int pass = 0;
    MG_TAIL_NODES(n) {  // b = P^T t_f
      double r = 0.0;
      if (id < n) {
#pragma unroll
        for (int k = 0; k < 3; ++k) {
          const int s2 = q + 4 * k;
          if (s2 >= 12) break;
          const int f = v.rid[s2 * n + id];
          if (f < 0) continue;
          double t = 0.0;
          if (l == l0) {
#pragma unroll
            for (int p = 0; p < MGS_TAIL_P; ++p)
              if (p == pass) t = tg[p][k];
          } else {
            t = tf[f];
          }
          r += mg_rw(s2) * t;
        }
      }
      ++pass;
      r = hw_sum1<4>(r);
      if (q == 0 && id < n) v.b[id] = mgs_mask(r, v.dinv[id]);
    }
    __syncthreads();
    if (l == c) break;
    const double om = om_s[l];
    MG_TAIL_NODES(n) {  // t = b - A (omega D^-1 b)
      const double Av = mgs_tapply(v, id, [&](int k) -> double { return om * v.dinv[k] * v.b[k]; });
      if (q == 0 && id < n) v.t[id] = mgs_mask(v.b[id] - Av, v.dinv[id]);
    }
    __syncthreads();
  }
  {  // coarsest solve
    const STLevel v = mgs_tl(A, c);
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
      int cur = (A.nu_c - 1) % 2 == 0 ? 0 : 1;
      for (int i = threadIdx.x; i < nd; i += blockDim.x) bufs[cur][i] = om * v.dinv[i] * v.b[i];
      __syncthreads();
      for (int sw = 1; sw < A.nu_c; ++sw) {
        const double* in = bufs[cur];
        double* out = bufs[cur ^ 1];
        MG_TAIL_NODES(v.n) {
          const double Ax = mgs_tapply(v, id, [&](int k) -> double { return in[k]; });
          if (q == 0 && id < v.n) out[id] = in[id] + om * v.dinv[id] * (v.b[id] - Ax);
        }
        cur ^= 1;
        __syncthreads();
      }
    }
    if (l0 == c)
      for (int i = threadIdx.x; i < nd; i += blockDim.x) A.L[c].e[i] = v.e[i];
  }
  for (int l = c - 1; l >= l0; --l) {
    const STLevel v = mgs_tl(A, l), vc = mgs_tl(A, l + 1);
    const int n = v.n;
    const double om = om_s[l];
    MG_TAIL_NODES(n) {  // y = omega D^-1 b + P e_c (into t)
      double r = 0.0, cnt = 0.0;
      if (id < n) {
        const int k = v.pid[q * n + id];
        if (k >= 0) {
          r = vc.e[k];
          cnt = 1.0;
        }
      }
      r = hw_sum1<4>(r);
      cnt = hw_sum1<4>(cnt);
      if (q == 0 && id < n) v.t[id] = mgs_mask(om * v.dinv[id] * v.b[id] + r / cnt, v.dinv[id]);
    }
    __syncthreads();
    double* eout = (l == l0) ? A.L[l].e : v.e;
    MG_TAIL_NODES(n) {  // e = y + omega D^-1 (b - A y)
      const double Ay = mgs_tapply(v, id, [&](int k) -> double { return v.t[k]; });
      if (q == 0 && id < n) eout[id] = v.t[id] + om * v.dinv[id] * (v.b[id] - Ay);
    }
    __syncthreads();
  }
}

}  // namespace pfb
