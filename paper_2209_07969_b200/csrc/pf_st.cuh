// Phase-field PCG on an assembled stencil (L2-resident meshes).
//
// The phase-field Newton system of one staggered pass (reference pf.py evolution, K_dd =
// sum_g N b_g N^T w + Gc l grad N grad N^T) is linear in the solve: its coefficients b_g are fixed
// by launch_evo_prepare.  On meshes whose assembled rows fit in L2, assembling it once per solve
// (k_evo_stencil, one pass) and iterating on the 3x3 (+ slit-tip) stencil trades the
// matrix-free march's ~50 DFMA per cell and per-row bookkeeping for 10 loads and 10 FMA per node.
// The rows are stored with D^-1 folded into the columns (S[s][i] = K(i, j) dinv(j), j = nbr[s][i])
// and zeroed on constrained rows, so w = A D^-1 r is one gather pass over r and needs no mask.
//
// k_cg_st is the single-reduction (Chronopoulos-Gear) Jacobi PCG of k_cg_sr (pf_cg.cuh) with the
// same stopping rule, iteration count semantics, warm start and result record, split into two
// node-parallel phases per iteration (update, then gather), each followed by a grid barrier.
namespace pfb {

#ifndef PFB_ST_U
#define PFB_ST_U 2
#endif
constexpr int ST_U = PFB_ST_U;  // nodes per thread per round of k_cg_st's phases
#ifndef PFB_ST_L1
#define PFB_ST_L1 1
#endif
// r gathers after the grid barrier: coherent L1-cached loads (the barrier's gpu-scope acquire
// invalidates L1, CCTL.IVALL, so plain loads observe the update phase's stores; the row's
// east/west/own values then come from L1) or, PFB_ST_L1=0, L2 loads (ld.cg).  cfg2 phase-field
// PCG iteration: 14.0 us (L1) / 14.7 us (L2) / 15.5 us matrix-free k_cg_sr<false>.
__device__ __forceinline__ double st_ld(const double* p) {
#if PFB_ST_L1
  return *p;
#else
  return __ldcg(p);
#endif
}

struct StArgs {
  const int* nbr;    // [MG_NS][n] stencil neighbours (pf_api.cu hl_stencil_ids of the fine layout)
  const int* ccell;  // [4][n] the cell in which node i is corner a (corner order of evo_cell_apply)
  const int* cslot;  // [4][n] stencil slot of corner b of that cell in bits 4b..4b+3 (15: none)
  double* S;         // [MG_NS][n] assembled rows, D^-1 folded into the columns
  int n;
};

// one thread per node: row i of K_dd from its (at most 4) cells, then the column scaling
__global__ void __launch_bounds__(256) k_evo_stencil(StArgs s, Consts C,
                                                     const double* __restrict__ b,
                                                     const double* __restrict__ dinv) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int n = s.n;
  if (i >= n) return;
  double acc[MG_NS];
#pragma unroll
  for (int t = 0; t < MG_NS; ++t) acc[t] = 0.0;
  if (__ldg(dinv + i) != 0.0) {
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      const int c = __ldg(s.ccell + (size_t)a * n + i);
      if (c < 0) continue;
      const unsigned sl = (unsigned)__ldg(s.cslot + (size_t)a * n + i);
      double bq[4];
      load4(b, c, bq);
      double t4[4];
#pragma unroll
      for (int g = 0; g < 4; ++g) t4[g] = C.Nw[g][a] * bq[g];
#pragma unroll
      for (int bb = 0; bb < 4; ++bb) {
        const double k = t4[0] * C.N[0][bb] + t4[1] * C.N[1][bb] + t4[2] * C.N[2][bb] +
                         t4[3] * C.N[3][bb] + C.lap[a][bb];
        const unsigned slot = (sl >> (4 * bb)) & 15u;
#pragma unroll
        for (int t = 0; t < MG_NS; ++t)
          if (slot == (unsigned)t) acc[t] += k;
      }
    }
  }
#pragma unroll
  for (int t = 0; t < MG_NS; ++t) {
    const int j = __ldg(s.nbr + (size_t)t * n + i);
    s.S[(size_t)t * n + i] = j >= 0 ? acc[t] * __ldg(dinv + j) : 0.0;
  }
}

// Vectors: x = a.x, r = a.r, w = A D^-1 r in a.q, s (= A p) in a.p0, p in a.p1.
//   pass 0:  (r.r, r.D^-1.r), w = A D^-1 r, w.D^-1.r
//   pass k:  s = w + beta s, p = D^-1 r + beta p, x += alpha p, r -= alpha s, then as pass 0
//   then     beta = g'/g, alpha = g'/(w.u - beta g'/alpha)      (k_cg_sr's recurrence)
#ifndef PFB_ST_MINB
#define PFB_ST_MINB 2
#endif
__global__ void __launch_bounds__(CG_NT, PFB_ST_MINB) k_cg_st(CgArgs a, StArgs st) {
  __shared__ CgSmem<false> S;
  cg::grid_group grid = cg::this_grid();
  double* part = a.partials;
  double bnorm_in = -1.0;
  if (a.n_guess > 0 && !a.probe) bnorm_in = warm_start<false>(a, S);
  const int n = st.n;
  const int i0 = blockIdx.x * blockDim.x + threadIdx.x, stride = gridDim.x * blockDim.x;
  const double* __restrict__ Sv = st.S;
  const int* __restrict__ nbr = st.nbr;
  long long k = 0;
  int status = CG_CONVERGED;
  double alpha = 0.0, beta = 0.0, gam = 0.0, rr = 0.0, bnorm = 0.0, atol = 0.0;
  for (;;) {
    double rrp = 0.0, gp = 0.0, dl = 0.0;
    // ST_U nodes per thread per round, every load of the round issued before the first use
    // (one L2 round trip per round instead of one per node)
    for (int base = i0; base < n; base += ST_U * stride) {  // update phase (owner-only)
      double di[ST_U], r[ST_U], w[ST_U], sv[ST_U], pv[ST_U], xv[ST_U];
#pragma unroll
      for (int u = 0; u < ST_U; ++u) {
        const int i = min(base + u * stride, n - 1);
        di[u] = __ldg(a.dinv + i);
        r[u] = __ldcg(a.r + i);
        if (k > 0) {
          w[u] = __ldcg(a.q + i);
          xv[u] = __ldcg(a.x + i);
          if (k > 1) {
            sv[u] = __ldcg(a.p0 + i);
            pv[u] = __ldcg(a.p1 + i);
          }
        }
      }
#pragma unroll
      for (int u = 0; u < ST_U; ++u) {
        const int i = base + u * stride;
        if (i >= n) continue;
        if (k > 0) {
          const double uu = di[u] * r[u];
          const double s2 = k == 1 ? w[u] : beta * sv[u] + w[u];
          const double p2 = k == 1 ? uu : beta * pv[u] + uu;
          a.p0[i] = s2;
          a.p1[i] = p2;
          a.x[i] = alpha * p2 + xv[u];
          r[u] = -alpha * s2 + r[u];
          a.r[i] = r[u];
        }
        if (node_owned(a.m, i)) {
          rrp += r[u] * r[u];
          gp += r[u] * (di[u] * r[u]);
        }
      }
    }
    grid.sync();
    for (int base = i0; base < n; base += ST_U * stride) {  // gather phase: w = A D^-1 r
      int j[ST_U][MG_NS];
      double c[ST_U][MG_NS];
#pragma unroll
      for (int u = 0; u < ST_U; ++u) {
        const int i = min(base + u * stride, n - 1);
#pragma unroll
        for (int t = 0; t < MG_NS; ++t) {
          j[u][t] = __ldg(nbr + (size_t)t * n + i);
          c[u][t] = __ldg(Sv + (size_t)t * n + i);
        }
      }
#pragma unroll
      for (int u = 0; u < ST_U; ++u) {
#pragma unroll
        for (int t = 0; t < MG_NS; ++t) c[u][t] *= j[u][t] >= 0 ? st_ld(a.r + j[u][t]) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < ST_U; ++u) {
        const int i = base + u * stride;
        if (i >= n) continue;
        double w = 0.0;
#pragma unroll
        for (int t = 0; t < MG_NS; ++t) w += c[u][t];
        a.q[i] = w;
        if (node_owned(a.m, i)) dl += w * (__ldg(a.dinv + i) * __ldcg(a.r + i));
      }
    }
    {
      double v[3] = {rrp, gp, dl};
      block_sum<3>(v, S.red);
      if (threadIdx.x == 0) {
        part[CG_PART_STRIDE * blockIdx.x] = v[0];
        part[CG_PART_STRIDE * blockIdx.x + 1] = v[1];
        part[CG_PART_STRIDE * blockIdx.x + 2] = v[2];
      }
    }
    grid.sync();
    double red[3];
    grid_reduce<3>(part, CG_PART_STRIDE, S.bc, red);
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
  if (status != CG_INDEFINITE && a.target) {
    for (int i = i0; i < n; i += stride) a.target[i] += __ldcg(a.x + i);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    a.result->iters = k;
    a.result->status = status;
    a.result->bnorm = bnorm;
    a.result->rnorm = sqrt(rr);
  }
}

}  // namespace pfb
