// pf_mgd.cuh — the multigrid PCG on row strips (multi-GPU).
//
// Each rank preconditions with its own V-cycle (pf_mg.cuh momentum / pf_mgs.cuh phase field) on
// the sub-mesh of its owned node rows, the ghost row above and (ranks > 0) the first owned row
// masked (homogeneous Dirichlet; the first owned row gets point Jacobi): a block-Jacobi
// preconditioner whose blocks are the strips, each solved approximately by one symmetric
// V(1,1)-cycle.  It is SPD, so the outer PCG -- the reference's Jacobi-PCG switch with
// M^-1 replaced (linsolve.py:48-54: x0 = 0, stop when ||r|| < rtol ||b||) -- keeps the solution
// contract; there is no coarse-grid exchange between GPUs (the hierarchies are local), the cost is
// a mild growth of the iteration count with the number of strips.  Per iteration: one local
// V-cycle (z), all-reduce of r.z, halo rows of z, one march p = z + beta p, q = A p over the local
// mesh (ghost rows included: every rank evaluates the ghost cells redundantly, pf_march.cuh),
// all-reduce of p.q, the streaming update of x and r, all-reduce of r.r.  Dot products sum owned
// nodes only (node_owned).
#pragma once

namespace pfb {

// dinv restricted to the V-cycle's nodes: owned, minus the strip's first owned node row
// [if_lo, if_hi) on ranks > 0 (the interface row, masked like the ghost row above, so every
// strip's local problem has a Dirichlet row: a strip with no physical Dirichlet boundary of its
// own, e.g. the upper L-panel strip, is not singular)
__global__ void k_mgd_mask(double* __restrict__ dst, const double* __restrict__ src, int comps,
                           DMesh m, int if_lo, int if_hi) {
  const long long n = (long long)comps * m.n_nodes;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const int node = (int)(i / comps);
    dst[i] = (node_owned(m, node) && !(node >= if_lo && node < if_hi)) ? src[i] : 0.0;
  }
}
// the interface row's block of the preconditioner: point Jacobi z = D^-1 r
__global__ void k_mgd_iface(double* __restrict__ z, const double* __restrict__ r,
                            const double* __restrict__ dinv, int comps, int if_lo, int if_hi) {
  const long long lo = (long long)comps * if_lo, n = (long long)comps * (if_hi - if_lo);
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    z[lo + i] = dinv[lo + i] * r[lo + i];
}
// partial sums of r.z over owned nodes (one per CTA)
__global__ void __launch_bounds__(MG_NT) k_mgd_dot(const double* __restrict__ r,
                                                    const double* __restrict__ z, int comps,
                                                    DMesh m, double* part) {
  __shared__ double red[MG_WARPS];
  const long long n = (long long)comps * m.n_nodes;
  double s = 0.0;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    if (node_owned(m, (int)(i / comps))) s += r[i] * z[i];
  double v[1] = {s};
  mg_block_sum<1>(v, red);
  if (threadIdx.x == 0) part[blockIdx.x] = v[0];
}

// x = 0; partial sums of r.r over owned nodes (one per CTA)
__global__ void __launch_bounds__(MG_NT) k_mgd_init(double* __restrict__ x,
                                                     const double* __restrict__ r, int comps,
                                                     DMesh m, double* part) {
  __shared__ double red[MG_WARPS];
  const long long n = (long long)comps * m.n_nodes;
  double rr = 0.0;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    x[i] = 0.0;
    const double v = r[i];
    if (node_owned(m, (int)(i / comps))) rr += v * v;
  }
  double v[1] = {rr};
  mg_block_sum<1>(v, red);
  if (threadIdx.x == 0) part[blockIdx.x] = v[0];
}

// global scalars (device, all-reduced): g[0] = r.z, g[1] = previous r.z, g[2] = p.q, g[3] = r.r
constexpr int MGD_RZ = 0, MGD_RZ_OLD = 1, MGD_PQ = 2, MGD_RR = 3;

// x += alpha p, r -= alpha q (alpha = r.z / p.q); partial sums of r.r over owned nodes
__global__ void __launch_bounds__(MG_NT) k_mgd_update(double* __restrict__ x,
                                                       double* __restrict__ r,
                                                       const double* __restrict__ p,
                                                       const double* __restrict__ q, int comps,
                                                       DMesh m, const double* g, double* part) {
  __shared__ double red[MG_WARPS];
  const double alpha = __ldcg(g + MGD_RZ) / __ldcg(g + MGD_PQ);
  const long long n = (long long)comps * m.n_nodes;
  double rr = 0.0;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    x[i] += alpha * p[i];
    const double v = r[i] - alpha * q[i];
    r[i] = v;
    if (node_owned(m, (int)(i / comps))) rr += v * v;
  }
  double v[1] = {rr};
  mg_block_sum<1>(v, red);
  if (threadIdx.x == 0) part[blockIdx.x] = v[0];
}

// p = z + beta p_old (beta = r.z / r.z_old; first: p = z), q = A p masked, p.q over owned nodes:
// the march of the full local mesh (PCG operator: the PCG's own inverse diagonal as the mask)
__global__ void __launch_bounds__(MG_NT, 2) k_mgd_dir_mom(MgArgs A, DMesh full, MarchGeom g,
                                                          const double* dinv, const double* gs,
                                                          int first, const double* pold,
                                                          double* pnew, double* part) {
  __shared__ MgWarp ws[MG_WARPS];
  __shared__ double red[MG_WARPS];
  const double beta = first ? 0.0 : __ldcg(gs + MGD_RZ) / __ldcg(gs + MGD_RZ_OLD);
  double pq = 0.0;
  FinePcg op{{&A.C, A.flags, A.d, dinv, A.phys, A.bq}, beta, A.z, first ? nullptr : pold, pnew,
             A.q, &pq, &full};
  const int w = blockIdx.x * MG_WARPS + (threadIdx.x >> 5);
  if (w < g.n_units) mg_march(full, g, w, op, ws[threadIdx.x >> 5]);
  double v[1] = {pq};
  mg_block_sum<1>(v, red);
  if (threadIdx.x == 0) part[blockIdx.x] = v[0];
}

__global__ void __launch_bounds__(MG_NT, 3) k_mgd_dir_pf(MgsArgs A, DMesh full, MarchGeom g,
                                                         const double* dinv, const double* gs,
                                                         int first, const double* pold,
                                                         double* pnew, double* part) {
  __shared__ MgWarp ws[MG_WARPS];
  __shared__ double red[MG_WARPS];
  const double beta = first ? 0.0 : __ldcg(gs + MGD_RZ) / __ldcg(gs + MGD_RZ_OLD);
  double pq = 0.0;
  SFinePcg op{{&A.C, A.bq, dinv}, beta, A.z, first ? nullptr : pold, pnew, A.q, &pq, &full};
  const int w = blockIdx.x * MG_WARPS + (threadIdx.x >> 5);
  if (w < g.n_units) mg_march(full, g, w, op, ws[threadIdx.x >> 5]);
  double v[1] = {pq};
  mg_block_sum<1>(v, red);
  if (threadIdx.x == 0) part[blockIdx.x] = v[0];
}

// g[RZ_OLD] = g[RZ] before the next r.z lands in g[RZ]
__global__ void k_mgd_shift(double* g) { g[MGD_RZ_OLD] = g[MGD_RZ]; }

}  // namespace pfb
