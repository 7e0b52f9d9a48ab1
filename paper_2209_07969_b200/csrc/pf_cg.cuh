// pf_cg.cuh — K4/K8 + K5 (+K10): persistent Jacobi-PCG, one cooperative launch per linear solve.
//
// Mirrors scipy.sparse.linalg.cg (SciPy 1.18.1, called at linsolve.py:51): x0 = 0, stop when the
// recursive residual satisfies ||r|| < rtol*||b||, z = D^-1 r, maxiter = 20 n, no breakdown test
// (the reference's bounded matrix keeps constrained components at zero, assembly.py:299-308,
// which the masked operator reproduces exactly).  Per iteration there are two grid barriers:
//   phase A (warp marching, pf_march.cuh): p_k = z_k + beta p_{k-1} evaluated on the fly for
//                    every node a warp touches (p double-buffered so neighbours read p_{k-1}
//                    while owners write p_k), q = A p_k (masked), partial p.q
//   phase B (flat):  r -= alpha q, x += alpha p_k, partials r.r and r.D^-1.r
// The SPD probe (K10, SURVEY.md §7 hard part 1) aborts at p.q <= 0.
//
// Phase A is the barrier-free warp march of pf_march.cuh (the first version of this kernel used
// 32x8 shared-memory tiles with three CTA barriers per tile; profiles/README.md has the history).
#pragma once
#include <type_traits>

namespace pfb {

#ifndef PFB_PHASEB_UNROLL
#define PFB_PHASEB_UNROLL 2
#endif
#ifndef PFB_CG_NT
#define PFB_CG_NT 256
#endif
constexpr int CG_NT = PFB_CG_NT;  // block size of the persistent PCG kernel
#ifndef PFB_CG_MINB_MOM
#define PFB_CG_MINB_MOM 2
#endif
#ifndef PFB_CG_MINB_EVO
#define PFB_CG_MINB_EVO 2
#endif

enum CgStatus { CG_CONVERGED = 0, CG_MAXITER = 1, CG_INDEFINITE = 2, CG_NAN = 3 };

struct CgResult {
  long long iters;
  int status;
  int pad;
  double bnorm, rnorm;
};

constexpr int WARM_MAX = 5;         // depth of the warm-start difference table
constexpr int CG_PART_STRIDE = 12;  // doubles per CTA in the partials buffer (warm start)
struct WarmTable {
  double* d[WARM_MAX];
};

struct MarchGeom {
  int n_strips, rows_per_unit, n_row_blocks, n_units;
};

struct CgArgs {
  DMesh m;
  Consts C;
  int vec2;             // 1: momentum (double2 per node)
  MarchGeom g;          // warp work units of the marching phase A (pf_march.cuh)
  long long ndof;        // flat length (2*n_nodes or n_nodes)
  const double* d;       // momentum: nodal d
  const uint8_t* flags;  // momentum: per-element tangent branch bits
  const double* b;       // phase field: [n_elems*4] Newton coefficient
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
  int probe;
  // optional warm start: backward-difference table of the last n_guess <= WARM_MAX solutions
  // (guess[0] = newest, guess[k] = k-th difference); x0 = their energy-optimal combination
  const double* guess[WARM_MAX];
  int n_guess;
  // single-reduction PCG (k_cg_sr) extra vectors: second r and w buffers, search direction
  double* r1;
  double* w1;
  double* pc;
};

template <bool MOM>
struct Node;
template <>
struct Node<true> {
  using T = double2;
  __device__ static T zero() { return make_double2(0.0, 0.0); }
  __device__ static T ld_cg(const double* p, int id) {
    return __ldcg(reinterpret_cast<const double2*>(p) + id);
  }
  __device__ static T ld_ro(const double* p, int id) {
    return __ldg(reinterpret_cast<const double2*>(p) + id);
  }
  __device__ static void st(double* p, int id, T v) { reinterpret_cast<double2*>(p)[id] = v; }
  __device__ static T mul(T a, T b) { return make_double2(a.x * b.x, a.y * b.y); }
  __device__ static T axpy(double s, T x, T y) { return make_double2(s * x.x + y.x, s * x.y + y.y); }
  __device__ static T mask(T v, T di) {
    return make_double2(di.x != 0.0 ? v.x : 0.0, di.y != 0.0 ? v.y : 0.0);
  }
  __device__ static unsigned freebits(T di) { return (di.x != 0.0 ? 1u : 0u) | (di.y != 0.0 ? 2u : 0u); }
  __device__ static T maskb(T v, unsigned b) {
    return make_double2((b & 1u) ? v.x : 0.0, (b & 2u) ? v.y : 0.0);
  }
  __device__ static double dot(T a, T b) { return a.x * b.x + a.y * b.y; }
};
template <>
struct Node<false> {
  using T = double;
  __device__ static T zero() { return 0.0; }
  __device__ static T ld_cg(const double* p, int id) { return __ldcg(p + id); }
  __device__ static T ld_ro(const double* p, int id) { return __ldg(p + id); }
  __device__ static void st(double* p, int id, T v) { p[id] = v; }
  __device__ static T mul(T a, T b) { return a * b; }
  __device__ static T axpy(double s, T x, T y) { return s * x + y; }
  __device__ static T mask(T v, T di) { return di != 0.0 ? v : 0.0; }
  __device__ static unsigned freebits(T di) { return di != 0.0 ? 1u : 0u; }
  __device__ static T maskb(T v, unsigned b) { return (b & 1u) ? v : 0.0; }
  __device__ static double dot(T a, T b) { return a * b; }
};

// ---------------------------------------------------------------------------------------
// phase-field element operator: (sum_g N b N^T w + grad_w L) p_e
__device__ __forceinline__ void evo_cell_apply(const Consts& C, const double (&pc)[4],
                                               const double (&bq)[4], double (&f)[4]) {
  double t4[4];
#pragma unroll
  for (int g = 0; g < 4; ++g)
    t4[g] = bq[g] * (C.N[g][0] * pc[0] + C.N[g][1] * pc[1] + C.N[g][2] * pc[2] +
                     C.N[g][3] * pc[3]);
#pragma unroll
  for (int aa = 0; aa < 4; ++aa)
    f[aa] = C.Nw[0][aa] * t4[0] + C.Nw[1][aa] * t4[1] + C.Nw[2][aa] * t4[2] +
            C.Nw[3][aa] * t4[3] + C.lap[aa][0] * pc[0] + C.lap[aa][1] * pc[1] +
            C.lap[aa][2] * pc[2] + C.lap[aa][3] * pc[3];
}

// One pass of the single-reduction (Chronopoulos-Gear) PCG, k_cg_sr: the march applies, at
// every node it touches, the previous iteration's updates s = w + beta s, r -= alpha s (and, at
// owned nodes, p = D^-1 r_old + beta p, x += alpha p), then multiplies u = D^-1 r.  r, s and w
// are ping-ponged (compile-time parity ODD, buffers straight from the kernel parameters)
// because neighbouring warps read a node's old values while its owner writes the new ones; p
// (CgArgs::pc) and x are read and written by the owner only.
template <bool ODD>
struct SrBuf {  // pass parity ODD reads the "in" buffers, writes the "out" buffers
  __device__ static const double* rin(const CgArgs& a) { return ODD ? a.r1 : a.r; }
  __device__ static double* rout(const CgArgs& a) { return ODD ? a.r : a.r1; }
  __device__ static const double* win(const CgArgs& a) { return ODD ? a.w1 : a.q; }
  __device__ static double* wout(const CgArgs& a) { return ODD ? a.q : a.w1; }
  __device__ static const double* sin(const CgArgs& a) { return ODD ? a.p1 : a.p0; }
  __device__ static double* sout(const CgArgs& a) { return ODD ? a.p0 : a.p1; }
};
struct SrScal {
  double alpha, beta;
  int first;  // pass 0: no update (u = D^-1 r0)
  int fresh;  // pass 1: no previous p, s
};

}  // namespace pfb
#include "pf_march.cuh"
namespace pfb {

// partial k of CTA i lives at part[stride*i + k]; every CTA sums in the same fixed order
template <int NV>
__device__ __forceinline__ void grid_reduce(const double* part, int stride, double* bc,
                                            double (&out)[NV]) {
  if (threadIdx.x < 32) {
    double s[NV];
#pragma unroll
    for (int k = 0; k < NV; ++k) s[k] = 0.0;
    lane_ordered_sum<NV>(part, stride, (int)gridDim.x, s);
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

// flat pass over double2 pairs: r -= alpha q and, XU, x += alpha p_k (update), partials r.r
// and r.D^-1.r.  The persistent kernel passes XU = false: its march applies the x update one
// iteration late (march_unit XUPD).
template <bool XU>
__device__ __forceinline__ void phase_b(const CgArgs& a, double alpha, const double* pk,
                                        bool update, double& rr, double& rz) {
  constexpr int U = PFB_PHASEB_UNROLL;
  const long long n2 = a.ndof >> 1;
  const long long stride = (long long)gridDim.x * blockDim.x;
  double2* r2 = reinterpret_cast<double2*>(a.r);
  double2* x2 = reinterpret_cast<double2*>(a.x);
  const double2* q2 = reinterpret_cast<const double2*>(a.q);
  const double2* p2 = reinterpret_cast<const double2*>(pk);
  const double2* d2 = reinterpret_cast<const double2*>(a.dinv);
  for (long long base = (long long)blockIdx.x * blockDim.x + threadIdx.x; base < n2;
       base += U * stride) {
    // loads are issued unconditionally (clamped index) so the unrolled arrays stay in registers
    double2 rv[U], qv[U], dv[U], pv[U], xv[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const long long i = min(base + u * stride, n2 - 1);
      rv[u] = __ldcg(r2 + i);
      dv[u] = __ldg(d2 + i);
      if (update) {
        qv[u] = __ldcg(q2 + i);
        if (XU) {
          pv[u] = __ldcg(p2 + i);
          xv[u] = __ldcg(x2 + i);
        }
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const long long i = base + u * stride;
      if (i < n2) {
        if (update) {
          rv[u].x -= alpha * qv[u].x;
          rv[u].y -= alpha * qv[u].y;
          r2[i] = rv[u];
          if (XU) {
            xv[u].x += alpha * pv[u].x;
            xv[u].y += alpha * pv[u].y;
            x2[i] = xv[u];
          }
        }
        // pair i holds node i (momentum) or nodes 2i, 2i+1 (phase field); ghosts do not count
        const bool o0 = node_owned(a.m, a.vec2 ? (int)i : (int)(2 * i));
        const bool o1 = a.vec2 ? o0 : node_owned(a.m, (int)(2 * i + 1));
        if (o0) {
          rr += rv[u].x * rv[u].x;
          rz += rv[u].x * (dv[u].x * rv[u].x);
        }
        if (o1) {
          rr += rv[u].y * rv[u].y;
          rz += rv[u].y * (dv[u].y * rv[u].y);
        }
      }
    }
  }
  if ((a.ndof & 1) && blockIdx.x == 0 && threadIdx.x == 0) {
    const long long i = a.ndof - 1;
    double rv = __ldcg(a.r + i);
    if (update) {
      rv -= alpha * __ldcg(a.q + i);
      a.r[i] = rv;
      if (XU) a.x[i] = __ldcg(a.x + i) + alpha * __ldcg(pk + i);
    }
    if (node_owned(a.m, (int)i)) {
      rr += rv * rv;
      rz += rv * (__ldg(a.dinv + i) * rv);
    }
  }
}

template <bool MOM>
struct CgSmem {
  DupRow<MOM> dup[CG_NT / 32];
  double red[CG_NT / 32 * CG_PART_STRIDE];
  double bc[CG_PART_STRIDE];
  double gram[WARM_MAX * WARM_MAX + WARM_MAX + 1];  // warm start: G, U^T b, b.b
};


// Galerkin warm start.  The host keeps, per kind of Newton system, the backward-difference
// table u_1 = v_1, u_2 = v_1 - v_2, u_3 = u_2(v_1,v_2) - u_2(v_2,v_3), ... of its last m
// solutions (k_warm_push).  Differences of consecutive solutions (which agree to ~1e-6) carry
// the trend at full relative precision, so the coefficients below stay O(1).  x0 = U y with
// (U^T A U) y = U^T b is the A-norm-closest point of span(U) to the solution: never worse than
// x0 = 0.  Directions whose Cholesky pivot falls below 1e-6 of their diagonal are dropped.
// r0 = b - A x0 is then formed by one more operator application, so it is consistent with x0
// whatever y is.  Returns ||b||; x and r are set for the PCG loop (r = b on entry).
template <bool MOM>
__device__ __forceinline__ double warm_start(const CgArgs& a, CgSmem<MOM>& S) {
  cg::grid_group grid = cg::this_grid();
  constexpr int M = WARM_MAX;
  const int gwarp = blockIdx.x * (CG_NT / 32) + (threadIdx.x >> 5),
            nwarps = gridDim.x * (CG_NT / 32);
  const long long stride = (long long)gridDim.x * blockDim.x;
  const long long i0 = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  double* part = a.partials;
  const int m = a.n_guess < M ? a.n_guess : M;
  // column k of G = U^T (A u_k) (free rows only); with k = 0 also c = U^T b and b.b
#pragma unroll 1
  for (int k = 0; k < m; ++k) {
    const double* uk = a.guess[0];
#pragma unroll
    for (int t = 1; t < M; ++t)
      if (k == t) uk = a.guess[t];
    for (int u = gwarp; u < a.g.n_units; u += nwarps) {
      double dummy = 0.0;
      march_unit<MOM, true>(a, a.g, u, true, 0.0, uk, nullptr, dummy, S.dup[threadIdx.x >> 5]);
    }
    grid.sync();
    double acc[CG_PART_STRIDE];
#pragma unroll
    for (int t = 0; t < CG_PART_STRIDE; ++t) acc[t] = 0.0;
    for (long long i = i0; i < a.ndof; i += stride) {
      if (!node_owned(a.m, (int)(a.vec2 ? i >> 1 : i)) || __ldg(a.dinv + i) == 0.0) continue;
      const double qi = __ldcg(a.q + i), bi = k == 0 ? __ldcg(a.r + i) : 0.0;
#pragma unroll
      for (int j = 0; j < M; ++j) {
        if (j < m && (j <= k || k == 0)) {
          const double uj = __ldg(a.guess[j] + i);
          if (j <= k) acc[j] += uj * qi;
          if (k == 0) acc[M + j] += uj * bi;
        }
      }
      if (k == 0) acc[2 * M] += bi * bi;
    }
    block_sum<CG_PART_STRIDE>(acc, S.red);
    if (threadIdx.x == 0)
      for (int t = 0; t < CG_PART_STRIDE; ++t) part[CG_PART_STRIDE * blockIdx.x + t] = acc[t];
    grid.sync();
    double g[CG_PART_STRIDE];
    grid_reduce<CG_PART_STRIDE>(part, CG_PART_STRIDE, S.bc, g);
    if (threadIdx.x == 0) {
      for (int j = 0; j <= k; ++j) S.gram[j * M + k] = S.gram[k * M + j] = g[j];
      if (k == 0)
        for (int j = 0; j <= M; ++j) S.gram[M * M + j] = g[M + j];
    }
    grid.sync();  // partials and S.bc are reused by the next column
  }
  double G[M][M], c[M];
#pragma unroll
  for (int j = 0; j < M; ++j) {
    c[j] = j < m ? S.gram[M * M + j] : 0.0;
#pragma unroll
    for (int k = 0; k < M; ++k) G[j][k] = (j < m && k < m) ? S.gram[j * M + k] : 0.0;
  }
  const double bb = m > 0 ? S.gram[M * M + M] : 0.0;
  // pivot-dropping Cholesky G = L L^T (identical arithmetic in every thread, compile-time
  // bounds so the arrays stay in registers)
  double L[M][M], z[M], y[M];
  bool keep[M];
#pragma unroll
  for (int i = 0; i < M; ++i) {
#pragma unroll
    for (int j = 0; j < M; ++j) L[i][j] = 0.0;
  }
#pragma unroll
  for (int i = 0; i < M; ++i) {
    double d = G[i][i];
#pragma unroll
    for (int k = 0; k < i; ++k) d -= L[i][k] * L[i][k];
    keep[i] = i < m && G[i][i] > 0.0 && d > 1e-6 * G[i][i];
    const double lii = keep[i] ? sqrt(d) : 1.0;
    L[i][i] = keep[i] ? lii : 0.0;
#pragma unroll
    for (int j = i + 1; j < M; ++j) {
      double e = G[j][i];
#pragma unroll
      for (int k = 0; k < i; ++k) e -= L[j][k] * L[i][k];
      L[j][i] = keep[i] ? e / lii : 0.0;
    }
  }
#pragma unroll
  for (int i = 0; i < M; ++i) {
    double e = c[i];
#pragma unroll
    for (int k = 0; k < i; ++k) e -= L[i][k] * z[k];
    z[i] = keep[i] ? e / L[i][i] : 0.0;
  }
  bool any = false;
#pragma unroll
  for (int i = M - 1; i >= 0; --i) {
    double e = z[i];
#pragma unroll
    for (int k = i + 1; k < M; ++k) e -= L[k][i] * y[k];
    y[i] = keep[i] ? e / L[i][i] : 0.0;
    any = any || y[i] != 0.0;
  }
  if (any) {
    for (long long i = i0; i < a.ndof; i += stride) {  // x0 = U y on the free DOFs
      double xv = 0.0;
      if (__ldg(a.dinv + i) != 0.0) {
#pragma unroll
        for (int k = 0; k < M; ++k)
          if (k < m) xv += y[k] * __ldg(a.guess[k] + i);
      }
      a.x[i] = xv;
    }
    grid.sync();
    for (int u = gwarp; u < a.g.n_units; u += nwarps) {  // q = A x0
      double dummy = 0.0;
      march_unit<MOM, true>(a, a.g, u, true, 0.0, a.x, nullptr, dummy, S.dup[threadIdx.x >> 5]);
    }
    grid.sync();
    for (long long i = i0; i < a.ndof; i += stride)  // r0 = b - A x0 (constrained rows stay 0)
      if (__ldg(a.dinv + i) != 0.0) a.r[i] = __ldcg(a.r + i) - __ldcg(a.q + i);
  }
  grid.sync();
  return sqrt(bb);
}

// warm-start history update after a solve: the difference table (guess[0] = newest solution,
// guess[k] = k-th backward difference) absorbs x in place; n_valid = entries before the push
__global__ void k_warm_push(WarmTable t, int n_valid, int depth, const double* __restrict__ x,
                            long long n) {
  // two entries per thread (16-byte accesses; every array is a 16-byte-padded allocation)
  const long long n2 = (n + 1) >> 1;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n2;
       i += (long long)gridDim.x * blockDim.x) {
    double2 cur = reinterpret_cast<const double2*>(x)[i];
#pragma unroll
    for (int k = 0; k < WARM_MAX; ++k) {
      if (k >= depth) break;
      double2* tk = reinterpret_cast<double2*>(t.d[k]) + i;
      const double2 old = k < n_valid ? *tk : make_double2(0.0, 0.0);
      *tk = cur;
      if (k >= n_valid) break;
      cur = make_double2(cur.x - old.x, cur.y - old.y);
    }
  }
}

// XUPD: lazy x update inside the march (fewer bytes, longer march): chosen by the host for
// meshes whose working set is far beyond L2 (pf_api.cu create_impl)
template <bool MOM, bool XUPD>
__global__ void __launch_bounds__(CG_NT, MOM ? PFB_CG_MINB_MOM : PFB_CG_MINB_EVO) k_cg(CgArgs a) {
  __shared__ CgSmem<MOM> S;
  cg::grid_group grid = cg::this_grid();
  const int gwarp = blockIdx.x * (CG_NT / 32) + (threadIdx.x >> 5),
            nwarps = gridDim.x * (CG_NT / 32);
  double* part = a.partials;
  double bnorm_in = -1.0;
  // warm start (phase-field solves only without the SPD probe: the predicate needs the Krylov
  // sequence from x0 = 0 that was validated against check_spd)
  if (a.n_guess > 0 && !a.probe) bnorm_in = warm_start<MOM>(a, S);
  double rr = 0.0, rz = 0.0;
  phase_b<!XUPD>(a, 0.0, nullptr, false, rr, rz);  // ||r0||^2 and r0.D^-1.r0 (r = b on entry)
  {
    double v[2] = {rr, rz};
    block_sum<2>(v, S.red);
    if (threadIdx.x == 0) {
      part[CG_PART_STRIDE * blockIdx.x] = v[0];
      part[CG_PART_STRIDE * blockIdx.x + 1] = v[1];
    }
  }
  grid.sync();
  // slots: 0/1 = r.r, r.z; 2 = p.q.  Each slot is rewritten only after a grid barrier that
  // every CTA passes after reading it.
  double red[2];
  grid_reduce<2>(part, CG_PART_STRIDE, S.bc, red);
  rr = red[0];
  double rho = red[1];
  const double bnorm = bnorm_in >= 0.0 ? bnorm_in : sqrt(rr);  // scipy: rtol * ||b||
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
      for (int u = gwarp; u < a.g.n_units; u += nwarps) {
        march_unit<MOM, false, XUPD>(a, a.g, u, first, beta, pold, pnew, pq,
                                       S.dup[threadIdx.x >> 5], alpha);
      }
      {
        double v[1] = {pq};
        block_sum<1>(v, S.red);
        if (threadIdx.x == 0) part[CG_PART_STRIDE * blockIdx.x + 2] = v[0];
      }
      grid.sync();
      double pqr[1];
      grid_reduce<1>(part + 2, CG_PART_STRIDE, S.bc, pqr);
      if (a.probe && !(pqr[0] > 0.0)) { status = CG_INDEFINITE; k += 1; break; }
      alpha = rho / pqr[0];
      rho_prev = rho;
      rr = 0.0;
      rz = 0.0;
      phase_b<!XUPD>(a, alpha, pnew, true, rr, rz);
      {
        double v[2] = {rr, rz};
        block_sum<2>(v, S.red);
        if (threadIdx.x == 0) {
          part[CG_PART_STRIDE * blockIdx.x] = v[0];
          part[CG_PART_STRIDE * blockIdx.x + 1] = v[1];
        }
      }
      grid.sync();
      grid_reduce<2>(part, CG_PART_STRIDE, S.bc, red);
      rr = red[0];
      rho = red[1];
      ++k;
    }
  }
  const bool xlast = XUPD && k > 0;
  if (status != CG_INDEFINITE && (xlast || a.target)) {
    // the last iteration's x += alpha p_{k-1} (deferred by the lazy update), then target += x
    const double* plast = ((k - 1) & 1) ? a.p1 : a.p0;
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < a.ndof;
         i += stride) {
      double xv = __ldcg(a.x + i);
      if (xlast) {
        xv += alpha * __ldcg(plast + i);
        a.x[i] = xv;
      }
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

// Single-reduction (Chronopoulos-Gear) Jacobi-PCG, persistent and cooperative like k_cg: ONE
// march and ONE grid barrier per iteration (k_cg: march, barrier, stream, barrier).  Same
// preconditioner, x0 and stopping rule (SciPy: ||r|| < rtol ||b||, maxiter, r recursive); the
// iterates equal the Hestenes-Stiefel ones in exact arithmetic (scripts/cgcg_study.py: counts
// within +-2 and true residuals at the same 1e-12 level on the reference's momentum systems).
//   pass 0:  u = D^-1 r0, w = A u, (r.r, r.u, w.u)
//   pass k:  s = w + beta s, p = D^-1 r + beta p (owners), x += alpha p, r -= alpha s,
//            u = D^-1 r, w = A u, (r.r, r.u, w.u)     [fused in the march, SrBuf/SrScal]
//   then     beta = g'/g, alpha = g'/(w.u - beta g'/alpha)   (denominator = p.Ap: the probe)
template <bool MOM>
__global__ void __launch_bounds__(CG_NT, MOM ? PFB_CG_MINB_MOM : PFB_CG_MINB_EVO)
    k_cg_sr(CgArgs a) {
  __shared__ CgSmem<MOM> S;
  cg::grid_group grid = cg::this_grid();
  const int gwarp = blockIdx.x * (CG_NT / 32) + (threadIdx.x >> 5),
            nwarps = gridDim.x * (CG_NT / 32);
  double* part = a.partials;
  double bnorm_in = -1.0;
  if (a.n_guess > 0 && !a.probe) bnorm_in = warm_start<MOM>(a, S);
  SrScal sp;
  long long k = 0;
  int status = CG_CONVERGED;
  double alpha = 0.0, beta = 0.0, gam = 0.0, rr = 0.0, bnorm = 0.0, atol = 0.0;
  for (;;) {
    sp.alpha = alpha;
    sp.beta = beta;
    sp.first = k == 0;
    sp.fresh = k == 1;
    double dl = 0.0, rrp = 0.0, gp = 0.0;
    if (k & 1) {
      for (int u = gwarp; u < a.g.n_units; u += nwarps)
        march_unit<MOM, false, false, 2>(a, a.g, u, false, 0.0, nullptr, nullptr, dl,
                                         S.dup[threadIdx.x >> 5], 0.0, &sp, &rrp, &gp);
    } else {
      for (int u = gwarp; u < a.g.n_units; u += nwarps)
        march_unit<MOM, false, false, 1>(a, a.g, u, false, 0.0, nullptr, nullptr, dl,
                                         S.dup[threadIdx.x >> 5], 0.0, &sp, &rrp, &gp);
    }
    const int off = (k & 1) ? 3 : 0;  // alternate slot sets: a slot is rewritten two barriers on
    {
      double v[3] = {rrp, gp, dl};
      block_sum<3>(v, S.red);
      if (threadIdx.x == 0) {
        part[CG_PART_STRIDE * blockIdx.x + off] = v[0];
        part[CG_PART_STRIDE * blockIdx.x + off + 1] = v[1];
        part[CG_PART_STRIDE * blockIdx.x + off + 2] = v[2];
      }
    }
    grid.sync();
    double red[3];
    grid_reduce<3>(part + off, CG_PART_STRIDE, S.bc, red);
    rr = red[0];
    const double gnew = red[1], delta = red[2];
    if (k == 0) {
      bnorm = bnorm_in >= 0.0 ? bnorm_in : sqrt(rr);  // scipy: rtol * ||b||
      atol = a.rtol * bnorm;
      if (bnorm == 0.0) break;
    }
    const double rn = sqrt(rr);
    if (rn < atol) break;
    if (!(rn == rn)) { status = CG_NAN; break; }
    if (k >= a.maxiter) { status = CG_MAXITER; break; }
    beta = k == 0 ? 0.0 : gnew / gam;
    const double den = k == 0 ? delta : delta - beta * gnew / alpha;  // = p.Ap
    if (a.probe && !(den > 0.0)) { status = CG_INDEFINITE; k += 1; break; }
    alpha = gnew / den;
    gam = gnew;
    ++k;
  }
  if (status != CG_INDEFINITE && a.target) {  // x is complete: target += x
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < a.ndof;
         i += stride)
      a.target[i] += __ldcg(a.x + i);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    a.result->iters = k;
    a.result->status = status;
    a.result->bnorm = bnorm;
    a.result->rnorm = sqrt(rr);
  }
}

// y = A x (unmasked) at the current state: one warp per marching unit
template <bool MOM>
__global__ void __launch_bounds__(NT) k_apply(CgArgs a, const double* x) {
  __shared__ DupRow<MOM> dup[NT / 32];
  const int u = blockIdx.x * (NT / 32) + (threadIdx.x >> 5);
  double pq = 0.0;
  if (u < a.g.n_units)
    march_unit<MOM, true>(a, a.g, u, true, 0.0, x, nullptr, pq, dup[threadIdx.x >> 5]);
}

}  // namespace pfb

// =========================================================================================
// Split-phase PCG: the same iteration as k_cg, but phase A (march) and phase B (stream) are
// separate kernels chained in a CUDA graph of CG_CHUNK iterations, so each phase is compiled
// for its own register budget / occupancy.  Device-side control: every CTA re-reduces the
// previous phase's per-CTA partials in a fixed order (deterministic, no atomics), so all CTAs
// agree on alpha, beta and the stopping decision; the first CTA of the deciding kernel records
// the outcome in CgCtl and every later kernel of the chunk exits immediately.
namespace pfb {

constexpr int CG_SLOTS = 3;  // ring of partial buffers: iteration k uses slot k mod 3

struct CgCtl {
  long long k0;     // first iteration of the current chunk
  long long iters;  // final iteration count (valid when done)
  int done, status;
  double atol, bnorm, rnorm;
};

struct SplitArgs {
  CgArgs c;
  CgCtl* ctl;
  // distributed mode: per-phase results reduced and all-reduced outside the kernels into
  // gA[slot] (p.q) and gB[slot][2] (r.r, r.D^-1.r); slot CG_SLOTS of gB holds the initial b
  const double* gA;
  const double* gB;
  double* partA;    // [CG_SLOTS][gridA]        p.q
  double* partB;    // [CG_SLOTS + 1][gridB][2] r.r, r.D^-1.r (slot CG_SLOTS: initial b)
  int gridA, gridB;
};

__device__ __forceinline__ int slot_of(long long k) { return (int)(k % CG_SLOTS); }

template <int NV>
__device__ __forceinline__ void reduce_parts(const double* part, int n, double* bc,
                                             double (&out)[NV]) {
  if (threadIdx.x < 32) {
    double s[NV];
#pragma unroll
    for (int q = 0; q < NV; ++q) s[q] = 0.0;
    lane_ordered_sum<NV>(part, NV, n, s);
#pragma unroll
    for (int q = 0; q < NV; ++q) s[q] = warp_sum(s[q]);
    if (threadIdx.x == 0) {
#pragma unroll
      for (int q = 0; q < NV; ++q) bc[q] = s[q];
    }
  }
  __syncthreads();
#pragma unroll
  for (int q = 0; q < NV; ++q) out[q] = bc[q];
}

// initial reduction over r = b: ||b||^2 and b.D^-1.b
template <bool MOM>
__global__ void __launch_bounds__(NT) k_cg_init(SplitArgs s) {
  __shared__ double red[NT / 32 * 2];
  double rr = 0.0, rz = 0.0;
  phase_b<true>(s.c, 0.0, nullptr, false, rr, rz);
  double v[2] = {rr, rz};
  block_sum<2>(v, red);
  double* pb = s.partB + (size_t)CG_SLOTS * s.gridB * 2;
  if (threadIdx.x == 0) { pb[2 * blockIdx.x] = v[0]; pb[2 * blockIdx.x + 1] = v[1]; }
  if (blockIdx.x == 0 && threadIdx.x == 0) { s.ctl->done = 0; s.ctl->status = CG_CONVERGED; }
}

#ifndef PFB_CGA_MINB_MOM
#define PFB_CGA_MINB_MOM 2
#endif
template <bool MOM>
__global__ void __launch_bounds__(NT, MOM ? PFB_CGA_MINB_MOM : 3) k_cg_a(SplitArgs s, int klocal) {
  __shared__ double bc[4];
  __shared__ double red[NT / 32];
  __shared__ DupRow<MOM> dup[NT / 32];
  if (s.ctl->done) return;
  const long long k = s.ctl->k0 + klocal;
  const int sb = k == 0 ? CG_SLOTS : slot_of(k - 1);
  double cur[2];
  if (s.gB) {
    cur[0] = s.gB[2 * sb];
    cur[1] = s.gB[2 * sb + 1];
  } else {
    reduce_parts<2>(s.partB + (size_t)sb * s.gridB * 2, s.gridB, bc, cur);  // r.r, r.D^-1.r
  }
  const double rn = sqrt(cur[0]);
  double atol;
  if (k == 0) {
    atol = s.c.rtol * rn;
    if (blockIdx.x == 0 && threadIdx.x == 0) { s.ctl->atol = atol; s.ctl->bnorm = rn; }
  } else {
    atol = s.ctl->atol;
  }
  int status = -1;
  if (k == 0 && rn == 0.0) status = CG_CONVERGED;  // b = 0: x = 0 (scipy returns b)
  else if (rn < atol) status = CG_CONVERGED;
  else if (!(rn == rn)) status = CG_NAN;
  else if (k >= s.c.maxiter) status = CG_MAXITER;
  if (status >= 0) {
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      s.ctl->iters = k;
      s.ctl->status = status;
      s.ctl->rnorm = rn;
      __threadfence();
      s.ctl->done = 1;
    }
    return;
  }
  double beta = 0.0;
  if (k > 0) {
    const int sp = k == 1 ? CG_SLOTS : slot_of(k - 2);
    double prev[2];
    if (s.gB) {
      prev[1] = s.gB[2 * sp + 1];
    } else {
      __syncthreads();
      reduce_parts<2>(s.partB + (size_t)sp * s.gridB * 2, s.gridB, bc, prev);
    }
    beta = cur[1] / prev[1];
  }
  double* pnew = (k & 1) ? s.c.p1 : s.c.p0;
  const double* pold = (k & 1) ? s.c.p0 : s.c.p1;
  double pq = 0.0;
  const int nwarps = gridDim.x * (NT / 32);
  for (int u = blockIdx.x * (NT / 32) + (threadIdx.x >> 5); u < s.c.g.n_units; u += nwarps)
    march_unit<MOM, false>(s.c, s.c.g, u, k == 0, beta, pold, pnew, pq, dup[threadIdx.x >> 5]);
  double v[1] = {pq};
  block_sum<1>(v, red);
  if (threadIdx.x == 0) s.partA[(size_t)slot_of(k) * s.gridA + blockIdx.x] = v[0];
}

template <bool MOM>
__global__ void __launch_bounds__(NT) k_cg_b(SplitArgs s, int klocal) {
  __shared__ double bc[4];
  __shared__ double red[NT / 32 * 2];
  if (s.ctl->done) return;
  const long long k = s.ctl->k0 + klocal;
  double pqv[1], cur[2];
  const int sb = k == 0 ? CG_SLOTS : slot_of(k - 1);
  if (s.gA) {
    pqv[0] = s.gA[slot_of(k)];
    cur[0] = s.gB[2 * sb];
    cur[1] = s.gB[2 * sb + 1];
  } else {
    reduce_parts<1>(s.partA + (size_t)slot_of(k) * s.gridA, s.gridA, bc, pqv);
    __syncthreads();
    reduce_parts<2>(s.partB + (size_t)sb * s.gridB * 2, s.gridB, bc, cur);
  }
  if (s.c.probe && !(pqv[0] > 0.0)) {
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      s.ctl->iters = k + 1;
      s.ctl->status = CG_INDEFINITE;
      __threadfence();
      s.ctl->done = 1;
    }
    return;
  }
  const double alpha = cur[1] / pqv[0];
  const double* pk = (k & 1) ? s.c.p1 : s.c.p0;
  double rr = 0.0, rz = 0.0;
  phase_b<true>(s.c, alpha, pk, true, rr, rz);
  double v[2] = {rr, rz};
  block_sum<2>(v, red);
  double* pb = s.partB + (size_t)slot_of(k) * s.gridB * 2;
  if (threadIdx.x == 0) { pb[2 * blockIdx.x] = v[0]; pb[2 * blockIdx.x + 1] = v[1]; }
}

// end of a chunk: advance the iteration base
__global__ void k_cg_advance(CgCtl* ctl, int chunk) {
  if (!ctl->done) ctl->k0 += chunk;
}

// target += x after convergence
__global__ void k_cg_finish(double* target, const double* x, long long n) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    target[i] += x[i];
}

}  // namespace pfb
