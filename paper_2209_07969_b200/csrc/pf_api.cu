// pf_api.cu — C-ABI (include/pf_b200.h) and host orchestration of the staggered hot path.
//
// Control flow mirrors the reference driver exactly (schemes.py:192-392): the Newton and
// staggered loops run on the host and read back ONE scalar block per Newton iteration
// (residual norm, gate count, SPD flag) through mapped pinned memory; every linear solve is ONE
// cooperative persistent PCG launch (pf_kernels.cuh: k_cg) with device-side stopping, so no
// host round trip happens inside a solve.
#include <cuda_runtime.h>

#include <algorithm>
#include <array>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <thread>
#include <utility>
#include <vector>

#include "../../include/pf_b200.h"
#include "pf_kernels.cuh"
#include "pf_comm.h"

using pfb::CgResult;

// One multigrid PCG instance (pf_mg.cuh): the momentum solves (phys 0) and the phase-field
// solves without the SPD probe (phys 1, the scalar field embedded as the x component of a
// two-component system) each have their own hierarchy, buffers and graphs.
struct MgInst {
  bool on = false;
  pfb::MgArgs A{};
  int gf = 1, gflat = 1;            // fine-march grid, flat-kernel grid
  std::vector<int> gl;              // warp-item grid per level (row-chunk kernels)
  std::vector<int> gn;              // node-parallel grid per level (assembled form)
  std::vector<int> lpn;             // lanes per node of the level's node kernels (1 | 4 | 16)
  pfb::MgIn* in = nullptr;          // pinned per-solve inputs (copied to A.in before a solve)
  cudaGraphExec_t setup_exec = nullptr, solve_exec = nullptr;
  // hierarchy reuse: the coarse levels (Galerkin matrices, omegas) are a preconditioner only;
  // they are rebuilt when the iteration count drifts above the count right after the last
  // rebuild, when the Dirichlet set changes, or after max_age solves (PFB200_MG_REUSE=0:
  // rebuild at every solve).  The fine level always uses the current tangent.
  bool built = false, reuse = true, reuse_cap = false;
  long long ref_iters = 0, last_iters = 0;
  int age = 0, max_age = 64;
  long long setups = 0;
  int setup_kernels = 0, body_kernels = 0;  // kernel nodes per graph (launch accounting)
  bool fuse = true;  // fused down / up kernels on the half-warp levels (PFB200_MG_FUSE=0: off)
  bool rows = true;  // row-table kernels on the one-thread-per-node levels (PFB200_MG_ROWS=0)
  cudaGraphExec_t vcycle_exec = nullptr;  // row strips: one V-cycle z = M^-1 r (pf_mgd.cuh)
  int vcycle_kernels = 0;
};

// The native scalar phase-field multigrid PCG (pf_mgs.cuh): hierarchy rebuilt at every solve
// (the phase-field tangent changes strongly between Newton iterations), solved by a graph whose
// PCG loop is a device-side WHILE node.
struct MgsInst {
  bool on = false;
  pfb::MgsArgs A{};
  int gf = 1, gfr = 1, gflat = 1;  // fine-march grids (gfr: the residual march), flat grid
  std::vector<int> gl, gn, lpn;
  pfb::MgIn* in = nullptr;
  // setup graphs: MGS_POW power steps (fast: a slightly low lambda estimate, a slightly larger
  // omega, fewer iterations) and MG_POW steps (safe: the redo when a solve on the fast hierarchy
  // overruns its budget -- an underestimated lambda can make the smoother diverge)
  cudaGraphExec_t setup_exec = nullptr, setup_safe_exec = nullptr, solve_exec = nullptr;
  int setup_kernels_safe = 0;
  bool rows = true;  // row-table kernels on the one-thread-per-node levels (PFB200_MGS_ROWS=0: off)
  long long last_iters = 0, redos = 0;
  cudaGraphExec_t vcycle_exec = nullptr;  // row strips: one V-cycle z = M^-1 r (pf_mgd.cuh)
  int vcycle_kernels = 0;
  long long setups = 0;
  int setup_kernels = 0, body_kernels = 0;
  bool fuse = true;
};

struct pf_handle {
  double hx = 0.0, hy = 0.0;  // uniform cell size (node (i, j) at (i hx, j hy))
  int device = 0;
  cudaStream_t stream = nullptr;
  pfb::DMesh dm{};
  pfb::Consts C{};
  pf_config cfg{};
  pf_material mat{};
  int n_nodes = 0, n_elems = 0, nx = 0, ny = 0;
  std::vector<int> h_nlo, h_nhi, h_nst, h_elo, h_ehi, h_est;
  // device row tables and tiles
  int *d_nlo = nullptr, *d_nhi = nullptr, *d_nst = nullptr;
  int *d_elo = nullptr, *d_ehi = nullptr, *d_est = nullptr;
  int2* d_tiles = nullptr;
  int4 *d_nrow = nullptr, *d_erow = nullptr;
  int n_tiles = 0;
  // state
  double *u = nullptr, *d = nullptr, *dprev = nullptr;
  double *trp = nullptr, *dev2 = nullptr, *psi = nullptr, *psimax = nullptr;
  // momentum work
  double *Ru = nullptr, *ru = nullptr, *xu = nullptr, *qu = nullptr, *p0u = nullptr,
         *p1u = nullptr, *dinvu = nullptr, *diagu = nullptr;
  double *r1u = nullptr, *w1u = nullptr, *pcu = nullptr;  // single-reduction PCG (k_cg_sr)
  double *r1d = nullptr, *w1d = nullptr, *pcd = nullptr;
  uint8_t* flags = nullptr;
  uint8_t* umask = nullptr;
  // phase-field work
  double *Rd = nullptr, *rd = nullptr, *xd = nullptr, *qd = nullptr, *p0d = nullptr,
         *p1d = nullptr, *dinvd = nullptr, *diagd = nullptr, *b = nullptr;
  uint8_t* pmask = nullptr;
  // scratch
  double* partials = nullptr;
  double* scratch = nullptr;   // [n_elems*16] strain / gate / extra outputs
  long long* d_idx = nullptr;  // index list scratch (BC dofs, reaction nodes)
  size_t d_idx_cap = 0;
  double* flushbuf = nullptr;
  size_t flush_n = 0;
  CgResult* h_cgres = nullptr;  // mapped pinned
  CgResult* d_cgres = nullptr;
  double* h_scal = nullptr;     // mapped pinned scalars
  double* d_scal = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr, evs0 = nullptr, evs1 = nullptr;
  int cg_grid = 1, cg_grid_evo = 1, sm_count = 0;
  // warm starts of the momentum PCG: previous solution of the same kind of Newton system
  // slot 0: the load-increment pass; slot s (1..WARM_SLOTS-1): staggered pass s (the last
  // slot also serves later passes) -- the previous load step's solve at the same pass index
  // Each slot keeps the backward-difference table of its last warm_depth (<= pfb::WARM_MAX)
  // solutions; the PCG starts from their energy-optimal combination (pf_cg.cuh warm_start).
  static constexpr int WARM_SLOTS = 4;
  bool warm = true;
  bool trace = false;
  bool evo_march = false;      // k_evo_prepare as a warp march (big single-GPU meshes)
  pfb::MarchGeom geom_prep{};
  int parts_n = 0;             // partial triples written by the last prepare kernel (0: n_tiles)
  bool mgs_gated = true;  // gated (S1/S2/S3) phase-field solves by the scalar multigrid PCG with
                          // the SPD probe inside (PFB200_MGS_GATED=0: the Jacobi-PCG probe)
  // cfg2 load steps 4..13, Jacobi momentum PCG iterations: depth 1 69634, 3 52336, 4 52151,
  // 5 51805; MG bench (phase-field tables): depth 3 682, 5 538 phase-field iterations.  The
  // multigrid solves use the first MG_WARM = 3 entries.
  int warm_depth = 5;
  double* warm_buf[WARM_SLOTS][pfb::WARM_MAX] = {};
  int warm_n[WARM_SLOTS] = {};
  // phase-field solves without the SPD probe (no gated Gauss point, or ST): the same
  // difference tables, per staggered pass (1, 2, >= 3)
  static constexpr int WARM_SLOTS_D = 3;
  double* warm_d[WARM_SLOTS_D][pfb::WARM_MAX] = {};
  int warm_nd[WARM_SLOTS_D] = {};
  bool xupd_mom = false, xupd_evo = false;  // lazy-x PCG variants (k_cg<MOM, true>)
  double* stage = nullptr;  // pinned host staging buffer for state transfers
  size_t stage_cap = 0;     // doubles
  bool sr_mom = false;  // momentum solves by the single-reduction PCG (k_cg_sr<true>)
  bool sr_evo = false;  // phase-field solves without the SPD probe by k_cg_sr<false>
  bool sr_evo_now = false;       // the kernel choice of the current phase-field launch
  long long evo_last_iters = 0;  // PCG iterations of the last converged phase-field solve
  // phase-field solves on the assembled stencil (pf_st.cuh k_cg_st) where its rows fit in L2
  bool st_evo = false, st_evo_now = false;
  pfb::StArgs st{};
  int cg_grid_st = 1;
  size_t sr_smem_evo = 0;
  size_t sr_smem = 0;   // its dynamic shared memory (cp.async staging slots)
  pfb::MarchGeom geom_mom{}, geom_evo{}, geom_apply{};
  // split-phase PCG (pf_cg.cuh: k_cg_a / k_cg_b chained in CUDA graphs)
  bool split = false;
  int chunk = 32;
  pfb::MarchGeom geom_a_mom{}, geom_a_evo{};
  int gridA_mom = 1, gridA_evo = 1, gridB = 1;
  pfb::CgCtl* d_ctl = nullptr;
  pfb::CgCtl* h_ctl = nullptr;  // pinned
  double *partA = nullptr, *partB = nullptr;
  cudaGraphExec_t graphs[2][2] = {{nullptr, nullptr}, {nullptr, nullptr}};  // [mom][probe]
  // row-strip decomposition: communicator and device reduction buffers
  pfb::Comm* comm = nullptr;
  double* d_red = nullptr;  // [16] device scalars for all-reduces
  double* gA = nullptr;     // [CG_SLOTS]       global p.q
  double* gB = nullptr;     // [CG_SLOTS+1][2]  global r.r, r.D^-1.r
  cudaGraphExec_t dgraphs[2][2] = {{nullptr, nullptr}, {nullptr, nullptr}};  // dist chunks
  long long l2_bytes = 0;
  // geometric-multigrid PCG instances (momentum; phase field on large meshes)
  MgInst mgu, mgd;
  MgsInst mgs;  // scalar phase-field multigrid (default for the phase field on large meshes)
  // row strips: the multigrid PCG with strip-local V-cycles (pf_mgd.cuh).  The hierarchies live
  // on the sub-mesh of the owned node rows (local rows mgd_row0 ..), the ghost row above masked.
  int mgd_row0 = 0;
  double* d_mgd = nullptr;      // [8] all-reduced scalars (pfb::MGD_*)
  double* h_mgd = nullptr;      // pinned copy of r.r
  double* mgd_part = nullptr;   // per-CTA partials
  int mgd_gflat = 1, mgd_gdir_u = 1, mgd_gdir_d = 1;
  pfb::MarchGeom mgd_geom_u{}, mgd_geom_d{};
  std::vector<void*> mg_allocs;
  // cached masks
  std::vector<int64_t> cons_key, pins_key;
  bool umask_all_free = true, pmask_all_free = true;
  int64_t n_pinned = 0;
  // accounting of the current call
  pf_stats acc{};
  std::string err;
};

static const char* kVersion = "paper_2209_07969_b200 0.1 (sm_100a FP64 matrix-free PCG)";

// ------------------------------------------------------------------------------------------
#define PF_CUDA(expr)                                                                \
  do {                                                                               \
    cudaError_t e__ = (expr);                                                        \
    if (e__ != cudaSuccess) {                                                        \
      h->err = std::string("CUDA error: ") + cudaGetErrorString(e__) + " at " #expr; \
      return PF_ERR_CUDA;                                                            \
    }                                                                                \
  } while (0)

#define PF_TRY(expr)                   \
  do {                                 \
    pf_status s__ = (expr);            \
    if (s__ != PF_OK) return s__;      \
  } while (0)

static pf_status fail(pf_handle* h, pf_status s, const std::string& msg) {
  h->err = msg;
  return s;
}

static pf_status launched(pf_handle* h) {
  h->acc.launches += 1;
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(h, PF_ERR_CUDA, std::string("launch: ") + cudaGetErrorString(e));
  return PF_OK;
}

template <class T>
static pf_status dalloc(pf_handle* h, T** p, size_t n) {
  // padded to a 16-byte multiple: the staged marches' bulk copies of 8-byte arrays end on an even
  // element (pf_mg.cuh mg_march_st)
  const size_t bytes = (std::max<size_t>(n, 1) * sizeof(T) + 15) & ~size_t(15);
  PF_CUDA(cudaMalloc((void**)p, bytes));
  PF_CUDA(cudaMemsetAsync(*p, 0, bytes, h->stream));
  return PF_OK;
}

static double now_s() {
  using namespace std::chrono;
  return duration<double>(steady_clock::now().time_since_epoch()).count();
}

// ------------------------------------------------------------------------------------------
// constants (restating the reference's shape-function arithmetic, assembly.py:28-43,108-129)
static void build_consts(pf_handle* h, double hx, double hy) {
  pfb::Consts& C = h->C;
  const double c = 1.0 / std::sqrt(3.0);
  const double gp[4][2] = {{-c, -c}, {c, -c}, {c, c}, {-c, c}};
  double dNx[4][4], dNy[4][4];
  for (int g = 0; g < 4; ++g) {
    const double xi = gp[g][0], et = gp[g][1];
    C.N[g][0] = 0.25 * ((1 - xi) * (1 - et));
    C.N[g][1] = 0.25 * ((1 + xi) * (1 - et));
    C.N[g][2] = 0.25 * ((1 + xi) * (1 + et));
    C.N[g][3] = 0.25 * ((1 - xi) * (1 + et));
    const double sx[4] = {-(1 - et), (1 - et), (1 + et), -(1 + et)};
    const double sy[4] = {-(1 - xi), -(1 + xi), (1 + xi), (1 - xi)};
    for (int a = 0; a < 4; ++a) {
      dNx[g][a] = (2.0 / hx) * (0.25 * sx[a]);
      dNy[g][a] = (2.0 / hy) * (0.25 * sy[a]);
    }
  }
  const double w = (hx * 0.5) * (hy * 0.5);
  C.w = w;
  C.Px = (1.0 + c) / (2.0 * hx);
  C.Mx = (1.0 - c) / (2.0 * hx);
  C.Py = (1.0 + c) / (2.0 * hy);
  C.My = (1.0 - c) / (2.0 * hy);
  C.Pxw = C.Px * w;
  C.Mxw = C.Mx * w;
  C.Pyw = C.Py * w;
  C.Myw = C.My * w;
  C.P2xw = C.Px * C.Px * w;
  C.M2xw = C.Mx * C.Mx * w;
  C.P2yw = C.Py * C.Py * w;
  C.M2yw = C.My * C.My * w;
  const pf_material& m = h->mat;
  const double grad_w = 2.0 * m.g_c * m.length_l / m.c_w;
  for (int g = 0; g < 4; ++g)
    for (int a = 0; a < 4; ++a) C.Nw[g][a] = C.N[g][a] * w;
  for (int a = 0; a < 4; ++a)
    for (int bb = 0; bb < 4; ++bb) {
      double s = 0.0;
      for (int g = 0; g < 4; ++g) s += (dNx[g][a] * dNx[g][bb] + dNy[g][a] * dNy[g][bb]) * w;
      C.lap[a][bb] = grad_w * s;
    }
  C.mu = m.mu;
  C.k = m.bulk_k;
  C.two_mu = 2.0 * m.mu;
  C.mu43 = 2.0 * m.mu * (1.0 - 1.0 / 3.0);
  C.third = 1.0 / 3.0;
  C.eta = m.eta;
  C.gamma = m.gamma;
  C.src_base = m.g_c / (m.c_w * m.length_l);
  C.grad_w = grad_w;
  C.psi_crit = m.g_c / (m.c_w * m.length_l);
  C.d_cap = h->cfg.d_cap;
  C.at2 = m.at2;
}

// ------------------------------------------------------------------------------------------
extern "C" const char* pf_version(void) { return kVersion; }

extern "C" const char* pf_last_error(const pf_handle* h) { return h ? h->err.c_str() : "null handle"; }

extern "C" void pf_destroy(pf_handle* h) {
  if (!h) return;
  cudaSetDevice(h->device);
  void* ptrs[] = {h->d_nlo, h->d_nhi, h->d_nst, h->d_elo, h->d_ehi, h->d_est, h->d_tiles,
                  h->d_nrow, h->d_erow,
                  h->u, h->d, h->dprev, h->trp, h->dev2, h->psi, h->psimax,
                  h->Ru, h->ru, h->xu, h->qu, h->p0u, h->p1u, h->dinvu, h->diagu, h->flags,
                  h->r1u, h->w1u, h->pcu, h->r1d, h->w1d, h->pcd,
                  h->umask, h->Rd, h->rd, h->xd, h->qd, h->p0d, h->p1d, h->dinvd, h->diagd,
                  h->b, h->pmask, h->partials, h->scratch, h->d_idx, h->flushbuf};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  for (auto& row : h->warm_buf)
    for (double* p : row)
      if (p) cudaFree(p);
  for (auto& row : h->warm_d)
    for (double* p : row)
      if (p) cudaFree(p);
  for (void* p : h->mg_allocs)
    if (p) cudaFree(p);
  for (MgInst* M : {&h->mgu, &h->mgd}) {
    if (M->in) cudaFreeHost(M->in);
    if (M->setup_exec) cudaGraphExecDestroy(M->setup_exec);
    if (M->solve_exec) cudaGraphExecDestroy(M->solve_exec);
    if (M->vcycle_exec) cudaGraphExecDestroy(M->vcycle_exec);
  }
  if (h->mgs.vcycle_exec) cudaGraphExecDestroy(h->mgs.vcycle_exec);
  if (h->d_mgd) cudaFree(h->d_mgd);
  if (h->h_mgd) cudaFreeHost(h->h_mgd);
  if (h->mgd_part) cudaFree(h->mgd_part);
  if (h->mgs.in) cudaFreeHost(h->mgs.in);
  if (h->mgs.setup_exec) cudaGraphExecDestroy(h->mgs.setup_exec);
  if (h->mgs.setup_safe_exec) cudaGraphExecDestroy(h->mgs.setup_safe_exec);
  if (h->mgs.solve_exec) cudaGraphExecDestroy(h->mgs.solve_exec);
  if (h->stage) cudaFreeHost(h->stage);
  for (auto& row : h->graphs)
    for (auto& g : row)
      if (g) cudaGraphExecDestroy(g);
  for (auto& row : h->dgraphs)
    for (auto& g : row)
      if (g) cudaGraphExecDestroy(g);
  delete h->comm;
  if (h->d_red) cudaFree(h->d_red);
  if (h->gA) cudaFree(h->gA);
  if (h->gB) cudaFree(h->gB);
  if (h->d_ctl) cudaFree(h->d_ctl);
  if (h->partA) cudaFree(h->partA);
  if (h->partB) cudaFree(h->partB);
  if (h->h_ctl) cudaFreeHost(h->h_ctl);
  if (h->h_cgres) cudaFreeHost(h->h_cgres);
  if (h->h_scal) cudaFreeHost(h->h_scal);
  if (h->ev0) cudaEventDestroy(h->ev0);
  if (h->ev1) cudaEventDestroy(h->ev1);
  if (h->evs0) cudaEventDestroy(h->evs0);
  if (h->evs1) cudaEventDestroy(h->evs1);
  if (h->stream) cudaStreamDestroy(h->stream);
  delete h;
}

static pf_status validate_mesh(pf_handle* h, const pf_mesh* m) {
  if (m->nx < 1 || m->ny < 1 || m->ny > 65535 || !(m->hx > 0.0) || !(m->hy > 0.0))
    return fail(h, PF_ERR_INVALID, "mesh: need 1 <= nx, 1 <= ny <= 65535 and hx, hy > 0");
  if (m->n_nodes <= 0 || 2 * m->n_nodes >= (int64_t)INT32_MAX || m->n_elems <= 0 ||
      4 * m->n_elems >= (int64_t)INT32_MAX)
    return fail(h, PF_ERR_INVALID, "mesh: sizes out of range for 32-bit device indexing");
  int64_t nn = 0, ne = 0;
  for (int j = 0; j <= m->ny; ++j) {
    if (m->node_lo[j] < 0 || m->node_hi[j] > m->nx + 1 || m->node_hi[j] < m->node_lo[j])
      return fail(h, PF_ERR_INVALID, "mesh: bad node row range");
    if (m->node_hi[j] > m->node_lo[j] && m->node_start[j] != nn)
      return fail(h, PF_ERR_INVALID, "mesh: node rows are not row-major compact");
    nn += m->node_hi[j] - m->node_lo[j];
  }
  if (m->notch_row >= 0) {
    if (m->notch_row > m->ny || m->notch_lo < 0 || m->notch_hi <= m->notch_lo ||
        m->dup_start != nn)
      return fail(h, PF_ERR_INVALID, "mesh: bad notch description");
    nn += m->notch_hi - m->notch_lo;
  }
  if (nn != m->n_nodes) return fail(h, PF_ERR_INVALID, "mesh: node count mismatch");
  for (int j = 0; j < m->ny; ++j) {
    const int lo = m->elem_lo[j], hi = m->elem_hi[j];
    if (hi < lo) return fail(h, PF_ERR_INVALID, "mesh: bad cell row range");
    if (hi > lo) {
      if (m->elem_start[j] != ne) return fail(h, PF_ERR_INVALID, "mesh: cells not row-major compact");
      // every corner must exist
      if (lo < m->node_lo[j] || hi + 1 > m->node_hi[j] || lo < m->node_lo[j + 1] ||
          hi + 1 > m->node_hi[j + 1])
        return fail(h, PF_ERR_INVALID, "mesh: cell corner outside node rows");
    }
    ne += hi - lo;
  }
  if (ne != m->n_elems) return fail(h, PF_ERR_INVALID, "mesh: element count mismatch");
  return PF_OK;
}


// ------------------------------------------------------------------------------------------
// multigrid hierarchy (pf_mg.cuh): row-compact layouts of the 2x2-agglomerated levels
struct HostLevel {
  int nx = 0, ny = 0;
  std::vector<int> nlo, nhi, nst, elo, ehi, est;
  int notch_row = -1, notch_lo = 0, notch_hi = 0, dup_start = 0, n_nodes = 0, n_elems = 0;
};

// coarse layout of f (every 2x2 block of cells -> one cell, slit kept on its coarse row), or
// false when f does not agglomerate (odd extents, rows or slit off the even lines)
static bool mg_coarsen(const HostLevel& f, HostLevel& c) {
  if (f.nx % 2 || f.ny % 2 || f.nx < 4 || f.ny < 4) return false;
  c = HostLevel();
  c.nx = f.nx / 2;
  c.ny = f.ny / 2;
  c.elo.resize(c.ny); c.ehi.resize(c.ny); c.est.resize(c.ny);
  for (int J = 0; J < c.ny; ++J) {
    const int a = 2 * J, b = 2 * J + 1;
    if (f.elo[a] != f.elo[b] || f.ehi[a] != f.ehi[b] || f.elo[a] % 2 || f.ehi[a] % 2) return false;
    c.elo[J] = f.elo[a] / 2;
    c.ehi[J] = f.ehi[a] / 2;
  }
  c.nlo.resize(c.ny + 1); c.nhi.resize(c.ny + 1); c.nst.resize(c.ny + 1);
  int n = 0;
  for (int J = 0; J <= c.ny; ++J) {
    const int lo = f.nlo[2 * J], hi = f.nhi[2 * J];
    if (lo % 2 || (hi - 1) % 2) return false;
    c.nlo[J] = lo / 2;
    c.nhi[J] = (hi - 1) / 2 + 1;
    c.nst[J] = n;
    n += c.nhi[J] - c.nlo[J];
  }
  int e = 0;
  for (int J = 0; J < c.ny; ++J) {
    c.est[J] = e;
    e += c.ehi[J] - c.elo[J];
  }
  c.n_elems = e;
  if (f.notch_row >= 0) {
    if (f.notch_row % 2 || f.notch_lo % 2 || f.notch_hi % 2) return false;
    c.notch_row = f.notch_row / 2;
    c.notch_lo = f.notch_lo / 2;
    c.notch_hi = f.notch_hi / 2;
    c.dup_start = n;
    n += c.notch_hi - c.notch_lo;
  }
  c.n_nodes = n;
  // every coarse node row must cover the odd fine rows next to it (bilinear prolongation)
  for (int j = 1; j < f.ny; j += 2) {
    const int J0 = j / 2, J1 = J0 + 1;
    const int lo = std::max(c.nlo[J0], c.nlo[J1]) * 2, hi = (std::min(c.nhi[J0], c.nhi[J1]) - 1) * 2 + 1;
    if (f.nlo[j] < lo || f.nhi[j] > hi) return false;
  }
  return true;
}


// node id at grid (i, j); up: the slit row's duplicates as seen from the cells above
static int hl_node(const HostLevel& L, int i, int j, bool up) {
  if (j < 0 || j > L.ny || i < L.nlo[j] || i >= L.nhi[j]) return -1;
  if (up && j == L.notch_row && i >= L.notch_lo && i < L.notch_hi) return L.dup_start + (i - L.notch_lo);
  return L.nst[j] + (i - L.nlo[j]);
}
static bool hl_cell(const HostLevel& L, int ci, int cj) {
  return cj >= 0 && cj < L.ny && ci >= L.elo[cj] && ci < L.ehi[cj];
}
static bool hl_dup_pos(const HostLevel& L, int i, int j) {
  return L.notch_row >= 0 && j == L.notch_row && i >= L.notch_lo && i < L.notch_hi;
}
template <class F>
static void hl_for_nodes(const HostLevel& L, F&& f) {  // f(id, i, j, dup)
  for (int j = 0; j <= L.ny; ++j)
    for (int i = L.nlo[j]; i < L.nhi[j]; ++i) f(L.nst[j] + (i - L.nlo[j]), i, j, false);
  if (L.notch_row >= 0)
    for (int i = L.notch_lo; i < L.notch_hi; ++i) f(L.dup_start + (i - L.notch_lo), i, L.notch_row, true);
}

// Stencil neighbours of every node, slot-major ([MG_NS][n]; pf_mg.cuh): slots 0-2 row j-1,
// 3-5 row j, 6-8 row j+1 (columns i-1, i, i+1), each looked up the way the cells coupling the
// two nodes see them (bottom corners from above the slit, top corners from below); slot 9 =
// the second face of a slit-tip neighbour (the only node coupled to both faces of one grid
// position).  -1 = no coupling.
static std::vector<int> hl_stencil_ids(const HostLevel& L) {
  const size_t n = L.n_nodes;
  std::vector<int> ids(n * pfb::MG_NS, -1);
  hl_for_nodes(L, [&](int id, int i, int j, bool) {
    auto o = [&](int s) -> int& { return ids[(size_t)s * n + id]; };
    const bool below = hl_node(L, i, j, false) == id;
    const bool above = hl_node(L, i, j, true) == id;
    for (int a = -1; a <= 1; ++a) {
      if (below) o(1 + a) = hl_node(L, i + a, j - 1, true);
      if (above) o(7 + a) = hl_node(L, i + a, j + 1, false);
      const int nb = below ? hl_node(L, i + a, j, false) : -1;
      const int na = above ? hl_node(L, i + a, j, true) : -1;
      if (nb >= 0 && na >= 0 && nb != na) {
        o(4 + a) = nb;
        o(9) = na;
      } else {
        o(4 + a) = nb >= 0 ? nb : na;
      }
    }
  });
  return ids;
}

// Restriction lists of coarse level c from fine level f ([12][n_c]): slot (b+1)*3 + (a+1) =
// the fine node at (2I+a, 2J+b) that interpolates from this coarse node (the regular node, or
// the slit duplicate on the far side), slots 9-11 = a second fine node at (2I+a, 2J) when both
// faces interpolate from it (the coarse slit tip).  Weights follow from the slot.
static std::vector<int> hl_restrict_ids(const HostLevel& f, const HostLevel& c) {
  const size_t n = c.n_nodes;
  std::vector<int> ids(n * 12, -1);
  hl_for_nodes(c, [&](int id, int I, int J, bool up) {
    const bool dpos = hl_dup_pos(c, I, J);
    for (int b = -1; b <= 1; ++b)
      for (int a = -1; a <= 1; ++a) {
        const int i = 2 * I + a, j = 2 * J + b;
        const int fr = hl_node(f, i, j, false);
        if (fr < 0) continue;
        const bool s_reg = f.notch_row >= 0 && j > f.notch_row;
        const bool use_r = !dpos || s_reg == up;
        const bool has_d = hl_dup_pos(f, i, j);
        const bool use_d = has_d && (!dpos || up);
        const int fd = has_d ? f.dup_start + (i - f.notch_lo) : -1;
        const int s = (b + 1) * 3 + (a + 1);
        if (use_r && use_d) {
          ids[(size_t)s * n + id] = fr;
          ids[(size_t)(9 + a + 1) * n + id] = fd;
        } else if (use_r) {
          ids[(size_t)s * n + id] = fr;
        } else if (use_d) {
          ids[(size_t)s * n + id] = fd;
        }
      }
  });
  return ids;
}

// Prolongation lists of fine level f from coarse level c ([4][n_f]): the coarse nodes
// (I0,J0), (I1,J0), (I0,J1), (I1,J1) that node (i, j) interpolates from (distinct ones only;
// weight 1 / their count), seen from the node's side of the slit.
static std::vector<int> hl_prolong_ids(const HostLevel& f, const HostLevel& c) {
  const size_t n = f.n_nodes;
  std::vector<int> ids(n * 4, -1);
  hl_for_nodes(f, [&](int id, int i, int j, bool dup) {
    const bool up = dup || (f.notch_row >= 0 && j > f.notch_row);
    const int I0 = i >> 1, J0 = j >> 1, I1 = I0 + (i & 1), J1 = J0 + (j & 1);
    ids[0 * n + id] = hl_node(c, I0, J0, up);
    if (I1 != I0) ids[1 * n + id] = hl_node(c, I1, J0, up);
    if (J1 != J0) ids[2 * n + id] = hl_node(c, I0, J1, up);
    if (I1 != I0 && J1 != J0) ids[3 * n + id] = hl_node(c, I1, J1, up);
  });
  return ids;
}

// multigrid arrays are padded to 16-byte multiples (k_mg_tail stages them with TMA bulk copies)
template <class T>
static cudaError_t mg_alloc(pf_handle* h, T** p, size_t n) {
  const size_t bytes = (std::max<size_t>(n, 1) * sizeof(T) + 15) & ~size_t(15);
  cudaError_t e = cudaMalloc((void**)p, bytes);
  if (e == cudaSuccess) {
    h->mg_allocs.push_back((void*)*p);
    e = cudaMemset(*p, 0, bytes);
  }
  return e;
}

static pf_status mg_build_graphs(pf_handle* h, MgInst& M);

// Level 0 of a multigrid hierarchy: the whole mesh on one GPU; on a row strip the sub-mesh of
// the owned node rows (local rows mgd_row0 .. ny: the ghost row below and its cell row are left
// out, the ghost row above is masked by the V-cycle's inverse diagonal).  Node and cell ids stay
// the strip's local ids, so the hierarchy reads and writes the strip's own vectors.
static HostLevel hl_level0(const pf_handle* h) {
  const int rb = h->comm ? h->mgd_row0 : 0;
  HostLevel f;
  f.nx = h->nx; f.ny = h->ny - rb;
  f.nlo.assign(h->h_nlo.begin() + rb, h->h_nlo.end());
  f.nhi.assign(h->h_nhi.begin() + rb, h->h_nhi.end());
  f.nst.assign(h->h_nst.begin() + rb, h->h_nst.end());
  f.elo.assign(h->h_elo.begin() + rb, h->h_elo.end());
  f.ehi.assign(h->h_ehi.begin() + rb, h->h_ehi.end());
  f.est.assign(h->h_est.begin() + rb, h->h_est.end());
  f.notch_row = h->dm.notch_row >= 0 ? h->dm.notch_row - rb : -1;
  f.notch_lo = h->dm.notch_lo; f.notch_hi = h->dm.notch_hi;
  f.dup_start = h->dm.dup_start; f.n_nodes = h->n_nodes;
  f.n_elems = 0;
  for (int j = 0; j < f.ny; ++j) f.n_elems += f.ehi[j] - f.elo[j];
  return f;
}
static pfb::DMesh dm_level0(const pf_handle* h) {
  const int rb = h->comm ? h->mgd_row0 : 0;
  pfb::DMesh m = h->dm;
  if (rb == 0) return m;
  m.ny -= rb;
  m.nrow += rb; m.erow += rb;
  m.nlo += rb; m.nhi += rb; m.nst += rb; m.elo += rb; m.ehi += rb; m.est += rb;
  if (m.notch_row >= 0) m.notch_row -= rb;
  return m;
}

static HostLevel hl_fine(const pf_handle* h) {
  HostLevel f;
  f.nx = h->nx; f.ny = h->ny;
  f.nlo = h->h_nlo; f.nhi = h->h_nhi; f.nst = h->h_nst;
  f.elo = h->h_elo; f.ehi = h->h_ehi; f.est = h->h_est;
  f.notch_row = h->dm.notch_row; f.notch_lo = h->dm.notch_lo; f.notch_hi = h->dm.notch_hi;
  f.dup_start = h->dm.dup_start; f.n_nodes = h->n_nodes; f.n_elems = h->n_elems;
  return f;
}

// assembled-stencil tables of the fine layout (pf_st.cuh StArgs): neighbours, and for every
// node the cells it is a corner of with the stencil slot of each of their corners.  A cell sees
// the slit row's nodes from its own side (lower face from below, duplicates from above).
static pf_status st_setup(pf_handle* h) {
  const HostLevel f = hl_fine(h);
  const size_t n = f.n_nodes;
  const std::vector<int> nb = hl_stencil_ids(f);
  std::vector<int> cc(4 * n, -1), cs(4 * n, -1);
  static const int dx[4] = {0, 1, 1, 0}, dy[4] = {0, 0, 1, 1};  // evo_cell_apply corner order
  bool ok = true;
  hl_for_nodes(f, [&](int id, int i, int j, bool) {
    for (int a = 0; a < 4; ++a) {
      const int ci = i - dx[a], cj = j - dy[a];
      if (!hl_cell(f, ci, cj) || hl_node(f, i, j, cj == j) != id) continue;
      unsigned sl = 0;
      for (int b = 0; b < 4; ++b) {
        const int nbid = hl_node(f, ci + dx[b], cj + dy[b], dy[b] == 0);
        int slot = -1;
        for (int s = 0; s < pfb::MG_NS && nbid >= 0; ++s)
          if (nb[(size_t)s * n + id] == nbid) slot = s;
        if (slot < 0) ok = false;
        sl |= (unsigned)(slot < 0 ? 15 : slot) << (4 * b);
      }
      cc[(size_t)a * n + id] = f.est[cj] + (ci - f.elo[cj]);
      cs[(size_t)a * n + id] = (int)sl;
    }
  });
  if (!ok) return fail(h, PF_ERR_INVALID, "assembled phase-field stencil: corner without a slot");
  int *dnb = nullptr, *dcc = nullptr, *dcs = nullptr;
  if (mg_alloc(h, &dnb, nb.size()) != cudaSuccess || mg_alloc(h, &dcc, cc.size()) != cudaSuccess ||
      mg_alloc(h, &dcs, cs.size()) != cudaSuccess ||
      mg_alloc(h, &h->st.S, (size_t)pfb::MG_NS * n) != cudaSuccess)
    return fail(h, PF_ERR_CUDA, "assembled phase-field stencil allocation failed");
  PF_CUDA(cudaMemcpy(dnb, nb.data(), nb.size() * sizeof(int), cudaMemcpyHostToDevice));
  PF_CUDA(cudaMemcpy(dcc, cc.data(), cc.size() * sizeof(int), cudaMemcpyHostToDevice));
  PF_CUDA(cudaMemcpy(dcs, cs.data(), cs.size() * sizeof(int), cudaMemcpyHostToDevice));
  h->st.nbr = dnb;
  h->st.ccell = dcc;
  h->st.cslot = dcs;
  h->st.n = (int)n;
  return PF_OK;
}


static pf_status mg_setup(pf_handle* h, MgInst& M, int phys, int fine_resident_warps) {
  const char* fz = getenv("PFB200_MG_FUSE");
  M.fuse = !(fz && std::string(fz) == "0");
  const char* rz = getenv("PFB200_MG_ROWS");
  M.rows = !(rz && std::string(rz) == "0");

  const char* tl = getenv("PFB200_MG_TAIL");  // tail levels: at most this many nodes
  const int tail_nodes = tl ? std::max(0, atoi(tl)) : 1 << 30;
  const char* nc = getenv("PFB200_MG_NUC");
  const int nu_c = nc ? std::max(1, atoi(nc)) : 16;
  std::vector<HostLevel> lv(1, hl_level0(h));
  while ((int)lv.size() < pfb::MG_MAXL && 2 * lv.back().n_nodes > pfb::MG_DENSE_MAX) {
    HostLevel c;
    if (!mg_coarsen(lv.back(), c)) break;
    lv.push_back(std::move(c));
  }
  const int nl = (int)lv.size();
  if (nl < 2) return PF_OK;  // nothing to agglomerate: Jacobi PCG
  pfb::MgArgs& A = M.A;
  A = pfb::MgArgs{};
  A.C = h->C;
  A.n_levels = nl;
  A.dense = 2 * lv.back().n_nodes <= pfb::MG_DENSE_MAX;
  A.nu_c = nu_c;
  // tail: the coarsest levels whose assembled form (plus the dense inverse) fits the
  // single-CTA kernel's shared memory (PFB200_MG_TAIL_KB, default 220)
  const char* tk = getenv("PFB200_MG_TAIL_KB");
  const size_t budget = (size_t)(tk ? std::max(0, atoi(tk)) : 220) * 1024;
  auto level_bytes = [&](const HostLevel& L) -> size_t {  // assembled form, 16-B aligned arrays
    auto al = [](size_t b) { return (b + 15) & ~size_t(15); };
    const size_t n = L.n_nodes;
    return al(4 * pfb::MG_NS * n) + al(4 * 12 * n) + al(4 * 4 * n) + al(8 * 4 * pfb::MG_NS * n) +
           4 * al(16 * n);
  };
  const size_t ainv_bytes = A.dense ? 8 * (size_t)(2 * lv.back().n_nodes) * (2 * lv.back().n_nodes) : 0;
  int nt = nl;
  size_t used = ainv_bytes;
  // (the top tail level's restriction sources are pre-loaded in registers: at most
  // MG_TAIL_P passes of MG_TAIL_NT / 4 nodes)
  while (nt > 1 && lv[nt - 1].n_nodes <= std::min(tail_nodes, pfb::MG_TAIL_P * pfb::MG_TAIL_NT / 4) &&
         used + level_bytes(lv[nt - 1]) <= budget) {
    used += level_bytes(lv[nt - 1]);
    --nt;
  }
  A.n_tail = nt;  // nt == nl: no tail kernel (the coarsest level is solved by grid kernels)
  {
    size_t off = 0;
    auto take = [&](size_t bytes) { const size_t o = off; off += (bytes + 15) & ~size_t(15); return (int)o; };
    for (int l = nt; l < nl; ++l) {
      const size_t n = lv[l].n_nodes;
      pfb::MgTailSlot& t = A.ts[l];
      t.nbr = take(4 * pfb::MG_NS * n);
      t.rid = take(4 * 12 * n);
      t.pid = take(4 * 4 * n);
      t.S = take(8 * 4 * pfb::MG_NS * n);
      t.dinv = take(16 * n);
      t.b = take(16 * n);
      t.t = take(16 * n);
      t.e = take(16 * n);
    }
    A.ts_ainv = take(ainv_bytes);
    A.ts_bytes = (int)off;
    if (nt < nl && cudaFuncSetAttribute(pfb::k_mg_tail, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        A.ts_bytes) != cudaSuccess)
      return fail(h, PF_ERR_CUDA, "k_mg_tail shared memory");
  }
  auto oom = [&]() { return fail(h, PF_ERR_CUDA, "multigrid allocation failed"); };
  M.gl.assign(nl, 1);
  M.gn.assign(nl, 1);
  M.lpn.assign(nl, 16);
  int coarse_items = 0;
  for (int l = 0; l < nl; ++l) {
    const HostLevel& L = lv[l];
    pfb::MgLevel& ML = A.L[l];
    pfb::DMesh& dm = ML.m;
    if (l == 0) {
      dm = dm_level0(h);
    } else {
      std::vector<int4> nrow(L.ny + 1), erow(L.ny);
      for (int j = 0; j <= L.ny; ++j) nrow[j] = make_int4(L.nlo[j], L.nhi[j], L.nst[j], 0);
      for (int j = 0; j < L.ny; ++j) erow[j] = make_int4(L.elo[j], L.ehi[j], L.est[j], 0);
      int4 *dn = nullptr, *de = nullptr;
      if (mg_alloc(h, &dn, nrow.size()) != cudaSuccess || mg_alloc(h, &de, erow.size()) != cudaSuccess)
        return oom();
      cudaMemcpy(dn, nrow.data(), nrow.size() * sizeof(int4), cudaMemcpyHostToDevice);
      cudaMemcpy(de, erow.data(), erow.size() * sizeof(int4), cudaMemcpyHostToDevice);
      dm = pfb::DMesh{};
      dm.nx = L.nx; dm.ny = L.ny;
      dm.nrow = dn; dm.erow = de;
      dm.notch_row = L.notch_row; dm.notch_lo = L.notch_lo; dm.notch_hi = L.notch_hi;
      dm.dup_start = L.dup_start;
      dm.n_nodes = L.n_nodes; dm.n_elems = L.n_elems;
      dm.own_lo = 0; dm.own_hi = L.n_nodes; dm.dup_lo = L.n_nodes;
      dm.cell_lo = 0; dm.cell_hi = L.n_elems;
      if (mg_alloc(h, &ML.K, 64 * (size_t)L.n_elems) != cudaSuccess ||
          mg_alloc(h, &ML.dinv, 2 * (size_t)L.n_nodes) != cudaSuccess ||
          mg_alloc(h, &ML.b, 2 * (size_t)L.n_nodes) != cudaSuccess ||
          mg_alloc(h, &ML.e, 2 * (size_t)L.n_nodes) != cudaSuccess)
        return oom();
      ML.items = pfb::mg_items(L.nx, L.ny, L.notch_row >= 0);
      ML.item_off = coarse_items;  // set below, once lpn is known
      M.gl[l] = (ML.items + pfb::MG_WARPS - 1) / pfb::MG_WARPS;
      // small levels: a half-warp per node (all loads of a node in flight); large levels: a
      // thread per node (latency hidden by occupancy).  Threshold: the level's lanes stay within
      // a quarter of one wave of resident threads (measured against a full wave: cfg2 MG
      // iteration 127.7 -> 121.3 us in the bench, cfg4 273.8 -> 247.2 us, cfg3/cfg5 unchanged;
      // an eighth of a wave: 132.5 us).  PFB200_MG_WAVE_X scales it (A/B tests).
      const char* wx = getenv("PFB200_MG_WAVE_X");
      const long long wave = (long long)(2048.0 * h->sm_count * (wx ? atof(wx) : 0.25));
      M.lpn[l] = 16LL * L.n_nodes <= wave ? 16 : (4LL * L.n_nodes <= wave ? 4 : 1);
      ML.lpn = M.lpn[l];
      ML.item_off = coarse_items;  // power steps: lpn threads per node, warp-aligned per level
      coarse_items += (int)(((long long)M.lpn[l] * L.n_nodes + 31) / 32 * 32);
      M.gn[l] = std::max(1, std::min((int)((M.lpn[l] * (long long)L.n_nodes + pfb::MG_NT - 1) / pfb::MG_NT),
                                         16 * h->sm_count));
      {  // assembled-form index tables (static per handle)
        const std::vector<int> nb = hl_stencil_ids(L), rd = hl_restrict_ids(lv[l - 1], L);
        int *dnb = nullptr, *drd = nullptr;
        if (mg_alloc(h, &dnb, nb.size()) != cudaSuccess || mg_alloc(h, &drd, rd.size()) != cudaSuccess ||
            mg_alloc(h, &ML.S, (size_t)4 * pfb::MG_NS * L.n_nodes) != cudaSuccess ||
            mg_alloc(h, &ML.Sf, (size_t)4 * pfb::MG_NS * L.n_nodes) != cudaSuccess)
          return oom();
        cudaMemcpy(dnb, nb.data(), nb.size() * sizeof(int), cudaMemcpyHostToDevice);
        cudaMemcpy(drd, rd.data(), rd.size() * sizeof(int), cudaMemcpyHostToDevice);
        ML.nbr = dnb;
        ML.rid = drd;
        if (l + 1 < nl) {
          const std::vector<int> pd = hl_prolong_ids(L, lv[l + 1]);
          int* dpd = nullptr;
          if (mg_alloc(h, &dpd, pd.size()) != cudaSuccess) return oom();
          cudaMemcpy(dpd, pd.data(), pd.size() * sizeof(int), cudaMemcpyHostToDevice);
          ML.pid = dpd;
        }
      }
    }
    if (mg_alloc(h, &ML.t, 2 * (size_t)L.n_nodes) != cudaSuccess) return oom();
  }
  A.coarse_items = coarse_items;
  A.g0 = pfb::make_march_geom(h->nx, lv[0].ny, fine_resident_warps);
  M.gf = (A.g0.n_units + pfb::MG_WARPS - 1) / pfb::MG_WARPS;
  M.gflat = 2 * h->sm_count;
  if (mg_alloc(h, &A.z, 2 * (size_t)h->n_nodes) != cudaSuccess) return oom();
  A.phys = phys;
  const char* s32 = getenv("PFB200_MG_S32");  // "0": FP64 coarse stencils in the V-cycle
  for (int l = 0; l < nl; ++l) {
    A.L[l].scalar = phys == 1 ? 1 : 0;
    A.L[l].s32 = (s32 && std::string(s32) == "0") ? 0 : 1;
  }
  if (phys == 0 && h->comm) {  // strips: the V-cycle's own inverse diagonal, ghost rows masked
    if (mg_alloc(h, &A.L[0].dinv, 2 * (size_t)h->n_nodes) != cudaSuccess) return oom();
  } else if (phys == 0) {
    A.L[0].dinv = h->dinvu;
  } else {  // phase field: scalar vectors packed as (value, 0) per node (y dofs dead)
    double* dinv2 = nullptr;
    if (mg_alloc(h, &dinv2, 2 * (size_t)h->n_nodes) != cudaSuccess) return oom();
    A.L[0].dinv = dinv2;
  }
  A.L[0].e = A.z;
  const int ndc = 2 * lv.back().n_nodes;
  if (A.dense && mg_alloc(h, &A.Ainv, (size_t)ndc * ndc) != cudaSuccess) return oom();
  const size_t npart = std::max<size_t>(
      std::max<size_t>((size_t)2 * M.gf + M.gflat, (size_t)M.gflat * 2 * pfb::MG_MAXL),
      (size_t)pfb::MG_WP * M.gf + M.gflat);
  if (mg_alloc(h, &A.part, npart) != cudaSuccess || mg_alloc(h, &A.ctl, 1) != cudaSuccess)
    return oom();
  // per-solve inputs: written on the host (pinned), copied to the device before each solve
  if (cudaHostAlloc((void**)&M.in, sizeof(pfb::MgIn), cudaHostAllocDefault) != cudaSuccess)
    return oom();
  pfb::MgIn* din = nullptr;
  if (mg_alloc(h, &din, 1) != cudaSuccess) return oom();
  A.in = din;
  A.d = h->d;
  A.flags = h->flags;
  A.bq = h->b;
  if (phys == 0) {
    A.x = h->xu; A.r = h->ru; A.p0 = h->p0u; A.p1 = h->p1u; A.q = h->qu;
  } else {
    const size_t n2 = 2 * (size_t)h->n_nodes;
    if (mg_alloc(h, &A.x, n2) != cudaSuccess || mg_alloc(h, &A.r, n2) != cudaSuccess ||
        mg_alloc(h, &A.p0, n2) != cudaSuccess || mg_alloc(h, &A.p1, n2) != cudaSuccess ||
        mg_alloc(h, &A.q, n2) != cudaSuccess)
      return oom();
  }
  A.result = h->d_cgres;
  A.ndof = 2LL * h->n_nodes;
  if (getenv("PFB200_MG_TAILCLK")) {
    if (mg_alloc(h, &A.tclk, 32) != cudaSuccess) return oom();
  }
  PF_TRY(mg_build_graphs(h, M));
  M.on = true;
  return PF_OK;
}

// Two graphs per handle: the hierarchy setup (Galerkin levels, diagonals, power steps, omega,
// dense coarsest inverse) and the solve (init, WHILE {one PCG iteration}, finish).
static pf_status mg_build_graphs(pf_handle* h, MgInst& M) {
  pfb::MgArgs& A = M.A;
  const int nl = A.n_levels;
  cudaStream_t s = h->stream;
  // ---- setup graph
  {
    cudaGraph_t g = nullptr;
    PF_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
    for (int lc = 1; lc < nl; ++lc) {
      const int cells = A.L[lc].m.nx * A.L[lc].m.ny;
      pfb::k_mg_galerkin<<<(cells + pfb::MG_WARPS - 1) / pfb::MG_WARPS, pfb::MG_NT, 0, s>>>(A, lc);
      pfb::k_mg_stencil<<<M.gl[lc], pfb::MG_NT, 0, s>>>(A, lc);
    }
    if (A.dense) pfb::k_mg_dense<<<1, pfb::MG_NT, 0, s>>>(A);
    // power steps for lambda_max(D^-1 A_l) (PFB200_MG_POW, default MG_POW); the fine march and
    // the coarse grid levels as separate launches (one grid queued the coarse blocks behind the
    // fine march's)
    const char* pc = getenv("PFB200_MG_POW");
    const int npow = pc ? std::max(2, std::min(pfb::MG_POW, atoi(pc))) : pfb::MG_POW;
    const int cb = (A.coarse_items + pfb::MG_NT - 1) / pfb::MG_NT;
    M.setup_kernels = 2 * (nl - 1) + (A.dense ? 1 : 0) + npow * (cb > 0 ? 2 : 1) + 1;
    for (int k = 1; k <= npow; ++k) {
      pfb::k_mg_pow<<<M.gf, pfb::MG_NT, 0, s>>>(A, k, M.gf);
      if (cb > 0) pfb::k_mg_pow<<<cb, pfb::MG_NT, 0, s>>>(A, k, 0);
    }
    pfb::k_mg_lambda<<<M.gflat, pfb::MG_NT, 0, s>>>(A, npow);
    cudaError_t e = cudaStreamEndCapture(s, &g);
    if (e != cudaSuccess) return fail(h, PF_ERR_CUDA, std::string("MG setup capture: ") + cudaGetErrorString(e));
    e = cudaGraphInstantiate(&M.setup_exec, g, 0);
    cudaGraphDestroy(g);
    if (e != cudaSuccess) return fail(h, PF_ERR_CUDA, std::string("MG setup graph: ") + cudaGetErrorString(e));
  }
  // ---- solve graph: init -> WHILE (cond) { iteration } -> finish.  PFB200_MG_UNROLL=N (profiling
  // only): N unconditional iterations instead of the WHILE node, so ncu sees every kernel.
#define MG_NODE_KERNEL(K, l, ...)                                                   \
  do {                                                                              \
    if (M.lpn[l] == 16) pfb::K<16><<<M.gn[l], pfb::MG_NT, 0, s>>>(__VA_ARGS__); \
    else if (M.lpn[l] == 4) pfb::K<4><<<M.gn[l], pfb::MG_NT, 0, s>>>(__VA_ARGS__); \
    else pfb::K<1><<<M.gn[l], pfb::MG_NT, 0, s>>>(__VA_ARGS__);                     \
  } while (0)
  auto body_kernels = [&](const pfb::MgArgs& B, bool krylov = true) {
    const int c = nl - 1, top = std::min(B.n_tail, c);  // grid levels [1, top)
    pfb::k_mg_fine_resid<<<M.gf, pfb::MG_NT, 0, s>>>(B);
    for (int l = 1; l < top; ++l) {
      // fused down-sweep only on the smallest grid levels: it evaluates 12 restriction sources
      // per stencil slot (cfg2, ncu: 16.6 k nodes 13.7 us fused vs 11.8 split; <= 4.2 k nodes
      // 7.5 / 6.4 vs 7.8 / 6.9)
      if (M.lpn[l] == 16 && M.fuse && B.L[l].m.n_nodes <= 8192) {
        pfb::k_mg_sdown<16><<<M.gn[l], pfb::MG_NT, 0, s>>>(B, l);
      } else if (M.lpn[l] == 1 && M.rows && B.L[l].m.n_nodes >= (1 << 20)) {  // large levels: row-table ids (bitwise equal)
        pfb::k_mg_rrestrict<<<M.gl[l], pfb::MG_NT, 0, s>>>(B, l);
        pfb::k_mg_rresid<<<M.gl[l], pfb::MG_NT, 0, s>>>(B, l);
      } else {
        MG_NODE_KERNEL(k_mg_srestrict, l, B, l);
        MG_NODE_KERNEL(k_mg_sresid, l, B, l);
      }
    }
    if (B.n_tail < nl) {
      pfb::k_mg_tail<<<1, pfb::MG_TAIL_NT, B.ts_bytes, s>>>(B);
    } else {  // coarsest level on the grid
      MG_NODE_KERNEL(k_mg_srestrict, c, B, c);
      if (B.dense) {
        pfb::k_mg_coarse_dense<<<1, pfb::MG_NT, 0, s>>>(B);
      } else {
        double* bufs[2] = {B.L[c].e, B.L[c].t};
        int cur = (B.nu_c - 1) % 2 == 0 ? 0 : 1;
        pfb::k_mg_jacobi0<<<M.gn[c], pfb::MG_NT, 0, s>>>(B, c, bufs[cur]);
        for (int k = 1; k < B.nu_c; ++k, cur ^= 1)
          MG_NODE_KERNEL(k_mg_ssweep, c, B, c, bufs[cur], bufs[cur ^ 1]);
      }
    }
    for (int l = top - 1; l >= 1; --l) {
      if (M.lpn[l] == 16 && M.fuse) {
        pfb::k_mg_sup<16><<<M.gn[l], pfb::MG_NT, 0, s>>>(B, l);
      } else if (M.lpn[l] == 1 && M.rows && B.L[l].m.n_nodes >= (1 << 20)) {
        // (the prolongation keeps its 16-byte index table: the row-table version measured slower)
        MG_NODE_KERNEL(k_mg_sprolongate, l, B, l);
        pfb::k_mg_rsmooth<<<M.gl[l], pfb::MG_NT, 0, s>>>(B, l);
      } else {
        MG_NODE_KERNEL(k_mg_sprolongate, l, B, l);
        MG_NODE_KERNEL(k_mg_ssmooth, l, B, l);
      }
    }
    pfb::k_mg_fine_smooth<<<M.gf, pfb::MG_NT, 0, s>>>(B);
    if (!krylov) return;
    pfb::k_mg_pcg<<<M.gf, pfb::MG_NT, 0, s>>>(B, M.gf);
    pfb::k_mg_update<<<M.gflat, pfb::MG_NT, 0, s>>>(B, M.gf, M.gf);
  };
  {
    const int c = nl - 1, top = std::min(A.n_tail, c);
    M.body_kernels = 1 + 3 + (A.n_tail < nl ? 1 : 1 + (A.dense ? 1 : A.nu_c));
    for (int l = 1; l < top; ++l) M.body_kernels += (M.lpn[l] == 16 && M.fuse) ? (A.L[l].m.n_nodes <= 8192 ? 2 : 3) : 4;
  }
  if (h->comm) {  // row strips: the preconditioner only, one V-cycle (pf_mgd.cuh drives the PCG)
    cudaGraph_t g = nullptr;
    A.use_cond = 0;
    PF_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
    body_kernels(A, false);
    PF_CUDA(cudaStreamEndCapture(s, &g));
    cudaError_t e = cudaGraphInstantiate(&M.vcycle_exec, g, 0);
    cudaGraphDestroy(g);
    if (e != cudaSuccess) return fail(h, PF_ERR_CUDA, std::string("MG V-cycle graph: ") + cudaGetErrorString(e));
    M.vcycle_kernels = M.body_kernels - 2;
    return PF_OK;
  }
  const char* un = getenv("PFB200_MG_UNROLL");
  const int unroll = un ? std::max(0, atoi(un)) : 0;
  if (unroll > 0) {
    cudaGraph_t g = nullptr;
    A.use_cond = 0;
    PF_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
    for (int k = 0; k < pfb::MG_WARM; ++k) pfb::k_mg_warm_q<<<M.gf, pfb::MG_NT, 0, s>>>(A, k);
    pfb::k_mg_init<<<M.gflat, pfb::MG_NT, 0, s>>>(A, M.gf);
    for (int it = 0; it < unroll; ++it) body_kernels(A);
    pfb::k_mg_finish<<<M.gflat, pfb::MG_NT, 0, s>>>(A);
    PF_CUDA(cudaStreamEndCapture(s, &g));
    cudaError_t e = cudaGraphInstantiate(&M.solve_exec, g, 0);
    cudaGraphDestroy(g);
    if (e != cudaSuccess) return fail(h, PF_ERR_CUDA, std::string("MG solve graph: ") + cudaGetErrorString(e));
    return PF_OK;
  }
  {
    cudaGraph_t g = nullptr;
    PF_CUDA(cudaGraphCreate(&g, 0));
    PF_CUDA(cudaGraphConditionalHandleCreate(&A.cond, g, 1, cudaGraphCondAssignDefault));
    A.use_cond = 1;
    cudaGraphNode_t n_init = nullptr, n_while = nullptr, n_fin = nullptr;
    {
      PF_CUDA(cudaStreamBeginCaptureToGraph(s, g, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
      for (int k = 0; k < pfb::MG_WARM; ++k) pfb::k_mg_warm_q<<<M.gf, pfb::MG_NT, 0, s>>>(A, k);
      pfb::k_mg_init<<<M.gflat, pfb::MG_NT, 0, s>>>(A, M.gf);
      cudaGraph_t gg = g;
      PF_CUDA(cudaStreamEndCapture(s, &gg));
      size_t nn = 0;
      PF_CUDA(cudaGraphGetNodes(g, nullptr, &nn));
      std::vector<cudaGraphNode_t> nodes(nn);
      PF_CUDA(cudaGraphGetNodes(g, nodes.data(), &nn));
      for (cudaGraphNode_t nd : nodes) {  // the WHILE node follows k_mg_init
        cudaKernelNodeParams kp{};
        if (cudaGraphKernelNodeGetParams(nd, &kp) == cudaSuccess && kp.func == (void*)pfb::k_mg_init)
          n_init = nd;
      }
      if (!n_init) return fail(h, PF_ERR_CUDA, "MG solve graph: init node not found");
    }
    cudaGraphNodeParams cp = {};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = A.cond;
    cp.conditional.type = cudaGraphCondTypeWhile;
    cp.conditional.size = 1;
    PF_CUDA(cudaGraphAddNode(&n_while, g, &n_init, 1, &cp));
    cudaGraph_t body = cp.conditional.phGraph_out[0];
    {
      PF_CUDA(cudaStreamBeginCaptureToGraph(s, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
      body_kernels(A);
      cudaGraph_t bb = body;
      PF_CUDA(cudaStreamEndCapture(s, &bb));
    }
    {
      cudaGraphNodeParams kp = {};
      kp.type = cudaGraphNodeTypeKernel;
      void* args[] = {&A};
      kp.kernel.func = (void*)pfb::k_mg_finish;
      kp.kernel.gridDim = dim3(M.gflat);
      kp.kernel.blockDim = dim3(pfb::MG_NT);
      kp.kernel.kernelParams = args;
      PF_CUDA(cudaGraphAddNode(&n_fin, g, &n_while, 1, &kp));
    }
    cudaError_t e = cudaGraphInstantiate(&M.solve_exec, g, 0);
    cudaGraphDestroy(g);
    if (e != cudaSuccess) return fail(h, PF_ERR_CUDA, std::string("MG solve graph: ") + cudaGetErrorString(e));
  }
  return PF_OK;
}

// ------------------------------------------------------------------------------------------
// native scalar phase-field multigrid (pf_mgs.cuh)
static pf_status mgs_build_graphs(pf_handle* h, MgsInst& M);

static pf_status mgs_setup(pf_handle* h, MgsInst& M, int fine_resident_warps) {
  const char* fz = getenv("PFB200_MG_FUSE");
  M.fuse = !(fz && std::string(fz) == "0");
  const char* rz = getenv("PFB200_MGS_ROWS");
  M.rows = !(rz && std::string(rz) == "0");
  const char* nc = getenv("PFB200_MG_NUC");
  const int nu_c = nc ? std::max(1, atoi(nc)) : 16;
  std::vector<HostLevel> lv(1, hl_level0(h));
  while ((int)lv.size() < pfb::MG_MAXL && lv.back().n_nodes > pfb::MGS_DENSE_MAX) {
    HostLevel c;
    if (!mg_coarsen(lv.back(), c)) break;
    lv.push_back(std::move(c));
  }
  const int nl = (int)lv.size();
  if (nl < 2) return PF_OK;
  pfb::MgsArgs& A = M.A;
  A = pfb::MgsArgs{};
  A.C = h->C;
  A.n_levels = nl;
  A.dense = lv.back().n_nodes <= pfb::MGS_DENSE_MAX;
  A.nu_c = nu_c;
  // tail: the coarsest levels whose assembled FP64 form fits the single-CTA kernel's shared
  // memory (PFB200_MG_TAIL_KB, default 220)
  const char* tk = getenv("PFB200_MG_TAIL_KB");
  const size_t budget = (size_t)(tk ? std::max(0, atoi(tk)) : 220) * 1024;
  auto al = [](size_t b) { return (b + 15) & ~size_t(15); };
  auto level_bytes = [&](const HostLevel& L) -> size_t {
    const size_t n = L.n_nodes;
    return al(4 * pfb::MG_NS * n) + al(4 * 12 * n) + al(4 * 4 * n) + al(8 * pfb::MG_NS * n) +
           4 * al(8 * n);
  };
  const size_t nc_nodes = lv.back().n_nodes;
  const size_t ainv_bytes = A.dense ? 8 * nc_nodes * nc_nodes : 0;
  int nt = nl;
  size_t used = ainv_bytes;
  while (nt > 1 && lv[nt - 1].n_nodes <= pfb::MGS_TAIL_P * pfb::MG_TAIL_NT / 4 &&
         used + level_bytes(lv[nt - 1]) <= budget) {
    used += level_bytes(lv[nt - 1]);
    --nt;
  }
  A.n_tail = nt;
  {
    size_t off = 0;
    auto take = [&](size_t bytes) { const size_t o = off; off += al(bytes); return (int)o; };
    for (int l = nt; l < nl; ++l) {
      const size_t n = lv[l].n_nodes;
      pfb::MgTailSlot& t = A.ts[l];
      t.nbr = take(4 * pfb::MG_NS * n);
      t.rid = take(4 * 12 * n);
      t.pid = take(4 * 4 * n);
      t.S = take(8 * pfb::MG_NS * n);
      t.dinv = take(8 * n);
      t.b = take(8 * n);
      t.t = take(8 * n);
      t.e = take(8 * n);
    }
    A.ts_ainv = take(ainv_bytes);
    A.ts_bytes = (int)off;
    if (nt < nl && cudaFuncSetAttribute(pfb::k_mgs_tail, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        A.ts_bytes) != cudaSuccess)
      return fail(h, PF_ERR_CUDA, "k_mgs_tail shared memory");
  }
  auto oom = [&]() { return fail(h, PF_ERR_CUDA, "phase-field multigrid allocation failed"); };
  M.gl.assign(nl, 1);
  M.gn.assign(nl, 1);
  M.lpn.assign(nl, 16);
  int coarse_items = 0;
  const long long wave = (long long)(2048.0 * h->sm_count * 0.25);
  for (int l = 0; l < nl; ++l) {
    const HostLevel& L = lv[l];
    pfb::MgsLevel& ML = A.L[l];
    pfb::DMesh& dm = ML.m;
    if (l == 0) {
      dm = dm_level0(h);
      ML.dinv = h->dinvd;
      if (h->comm && mg_alloc(h, &ML.dinv, (size_t)L.n_nodes) != cudaSuccess) return oom();
      if (mg_alloc(h, &ML.t, (size_t)L.n_nodes) != cudaSuccess) return oom();
      continue;
    }
    std::vector<int4> nrow(L.ny + 1), erow(L.ny);
    for (int j = 0; j <= L.ny; ++j) nrow[j] = make_int4(L.nlo[j], L.nhi[j], L.nst[j], 0);
    for (int j = 0; j < L.ny; ++j) erow[j] = make_int4(L.elo[j], L.ehi[j], L.est[j], 0);
    int4 *dn = nullptr, *de = nullptr;
    if (mg_alloc(h, &dn, nrow.size()) != cudaSuccess || mg_alloc(h, &de, erow.size()) != cudaSuccess)
      return oom();
    PF_CUDA(cudaMemcpy(dn, nrow.data(), nrow.size() * sizeof(int4), cudaMemcpyHostToDevice));
    PF_CUDA(cudaMemcpy(de, erow.data(), erow.size() * sizeof(int4), cudaMemcpyHostToDevice));
    dm = pfb::DMesh{};
    dm.nx = L.nx; dm.ny = L.ny;
    dm.nrow = dn; dm.erow = de;
    dm.notch_row = L.notch_row; dm.notch_lo = L.notch_lo; dm.notch_hi = L.notch_hi;
    dm.dup_start = L.dup_start;
    dm.n_nodes = L.n_nodes; dm.n_elems = L.n_elems;
    dm.own_lo = 0; dm.own_hi = L.n_nodes; dm.dup_lo = L.n_nodes;
    dm.cell_lo = 0; dm.cell_hi = L.n_elems;
    const size_t n = L.n_nodes;
    if (mg_alloc(h, &ML.K, 16 * (size_t)L.n_elems) != cudaSuccess ||
        mg_alloc(h, &ML.dinv, n) != cudaSuccess || mg_alloc(h, &ML.b, n) != cudaSuccess ||
        mg_alloc(h, &ML.e, n) != cudaSuccess || mg_alloc(h, &ML.t, n) != cudaSuccess)
      return oom();
    ML.items = pfb::mg_items(L.nx, L.ny, L.notch_row >= 0);
    M.gl[l] = (ML.items + pfb::MG_WARPS - 1) / pfb::MG_WARPS;
    M.lpn[l] = 16LL * L.n_nodes <= wave ? 16 : (4LL * L.n_nodes <= wave ? 4 : 1);
    ML.lpn = M.lpn[l];
    ML.in_tail = l >= nt ? 1 : 0;
    if (l < nt) {
      ML.item_off = coarse_items;
      coarse_items += (int)(((long long)M.lpn[l] * L.n_nodes + 31) / 32 * 32);
    }
    M.gn[l] = std::max(1, std::min((int)((M.lpn[l] * (long long)L.n_nodes + pfb::MG_NT - 1) / pfb::MG_NT),
                                   16 * h->sm_count));
    const std::vector<int> nb = hl_stencil_ids(L), rd = hl_restrict_ids(lv[l - 1], L);
    int *dnb = nullptr, *drd = nullptr;
    if (mg_alloc(h, &dnb, nb.size()) != cudaSuccess || mg_alloc(h, &drd, rd.size()) != cudaSuccess)
      return oom();
    if (l >= nt ? mg_alloc(h, &ML.S, (size_t)pfb::MG_NS * n) != cudaSuccess
                : mg_alloc(h, &ML.Sf, (size_t)pfb::MG_NS * n) != cudaSuccess)
      return oom();
    PF_CUDA(cudaMemcpy(dnb, nb.data(), nb.size() * sizeof(int), cudaMemcpyHostToDevice));
    PF_CUDA(cudaMemcpy(drd, rd.data(), rd.size() * sizeof(int), cudaMemcpyHostToDevice));
    ML.nbr = dnb;
    ML.rid = drd;
    if (l + 1 < nl) {
      const std::vector<int> pd = hl_prolong_ids(L, lv[l + 1]);
      int* dpd = nullptr;
      if (mg_alloc(h, &dpd, pd.size()) != cudaSuccess) return oom();
      PF_CUDA(cudaMemcpy(dpd, pd.data(), pd.size() * sizeof(int), cudaMemcpyHostToDevice));
      ML.pid = dpd;
    }
  }
  A.coarse_items = coarse_items;
  A.g0 = pfb::make_march_geom(h->nx, lv[0].ny, fine_resident_warps);
  M.gf = (A.g0.n_units + pfb::MG_WARPS - 1) / pfb::MG_WARPS;
  {
    int orr = 0;
    PF_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&orr, pfb::k_mgs_fine_resid, pfb::MG_NT, 0));
    A.g0r = pfb::make_march_geom(h->nx, lv[0].ny, std::max(1, orr) * h->sm_count * pfb::MG_WARPS);
    M.gfr = (A.g0r.n_units + pfb::MG_WARPS - 1) / pfb::MG_WARPS;
  }
  M.gflat = 2 * h->sm_count;
  const size_t nn = h->n_nodes;
  if (mg_alloc(h, &A.z, nn) != cudaSuccess) return oom();
  A.L[0].e = A.z;
  if (A.dense && mg_alloc(h, &A.Ainv, nc_nodes * nc_nodes) != cudaSuccess) return oom();
  const size_t npart = std::max<size_t>((size_t)2 * M.gf + M.gflat, (size_t)M.gflat * 2 * pfb::MG_MAXL);
  if (mg_alloc(h, &A.part, npart) != cudaSuccess || mg_alloc(h, &A.ctl, 1) != cudaSuccess)
    return oom();
  if (cudaHostAlloc((void**)&M.in, sizeof(pfb::MgIn), cudaHostAllocDefault) != cudaSuccess)
    return oom();
  *M.in = pfb::MgIn{};
  pfb::MgIn* din = nullptr;
  if (mg_alloc(h, &din, 1) != cudaSuccess) return oom();
  A.in = din;
  A.bq = h->b;
  // the phase-field Newton system in place: right-hand side rd (consumed), solution xd; the
  // Jacobi PCG's direction buffers serve as p and q
  A.r = h->rd;
  A.x = h->xd;
  A.p0 = h->p0d;
  A.p1 = h->p1d;
  A.q = h->qd;
  A.result = h->d_cgres;
  A.n = (long long)nn;
  PF_TRY(mgs_build_graphs(h, M));
  M.on = true;
  return PF_OK;
}

static pf_status mgs_build_graphs(pf_handle* h, MgsInst& M) {
  pfb::MgsArgs& A = M.A;
  const int nl = A.n_levels;
  cudaStream_t s = h->stream;
  // power steps from a hashed start at every setup: MGS_POW (PFB200_MGS_POW) and MG_POW (the safe
  // redo).  (Warm-started power steps from the previous setup's vectors were tried: the
  // phase-field iteration counts drifted up over the load steps at cfg5.)
  const char* pc = getenv("PFB200_MGS_POW");
  const int npow_fast = pc ? std::max(2, std::min(pfb::MG_POW, atoi(pc))) : pfb::MGS_POW;
  for (int safe = 0; safe < 2; ++safe) {
    const int npow = safe ? pfb::MG_POW : npow_fast;
    const bool warm = false;
    pfb::MgsArgs B = A;
    B.pow_warm = warm ? 1 : 0;
    cudaGraph_t g = nullptr;
    PF_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
    for (int lc = 1; lc < nl; ++lc) {
      const long long cells = (long long)B.L[lc].m.nx * B.L[lc].m.ny;
      const int gb = (int)std::max(1LL, std::min((cells + pfb::MG_NT - 1) / pfb::MG_NT,
                                                 64LL * h->sm_count));
      pfb::k_mgs_galerkin<<<gb, pfb::MG_NT, 0, s>>>(B, lc);
      pfb::k_mgs_stencil<<<M.gl[lc], pfb::MG_NT, 0, s>>>(B, lc);
    }
    if (B.dense) pfb::k_mgs_dense<<<1, pfb::MG_NT, 0, s>>>(B);
    // the fine march and the coarse grid levels of a power step as two launches: in one grid
    // the coarse blocks queued behind the fine march's (3.3 ms per step at cfg5)
    // the large one-thread-per-node levels (the first ones) by the row-table kernel
    int lr = 1;
    while (lr < B.n_tail && M.lpn[lr] == 1 && M.rows && B.L[lr].m.n_nodes >= (1 << 20)) ++lr;
    const int off0 = lr < B.n_tail ? B.L[lr].item_off : B.coarse_items;
    const int cb = (B.coarse_items - off0 + pfb::MG_NT - 1) / pfb::MG_NT;
    for (int k = 1; k <= npow; ++k) {
      pfb::k_mgs_pow<<<M.gf, pfb::MG_NT, 0, s>>>(B, k, M.gf);
      for (int l = 1; l < lr; ++l) pfb::k_mgs_rpow<<<M.gl[l], pfb::MG_NT, 0, s>>>(B, l, k);
      if (cb > 0) pfb::k_mgs_pow_coarse<<<cb, pfb::MG_NT, 0, s>>>(B, k, off0);
    }
    if (B.n_tail < nl) pfb::k_mgs_pow_tail<<<1, pfb::MG_TAIL_NT, 0, s>>>(B, npow);
    pfb::k_mgs_lambda<<<M.gflat, pfb::MG_NT, 0, s>>>(B, npow);
    const int nk = 2 * (nl - 1) + (B.dense ? 1 : 0) + npow * ((cb > 0 ? 2 : 1) + (lr - 1)) +
                   (B.n_tail < nl ? 1 : 0) + 1;
    (safe ? M.setup_kernels_safe : M.setup_kernels) = nk;
    cudaError_t e = cudaStreamEndCapture(s, &g);
    if (e != cudaSuccess) return fail(h, PF_ERR_CUDA, std::string("MGS setup capture: ") + cudaGetErrorString(e));
    e = cudaGraphInstantiate(safe ? &M.setup_safe_exec : &M.setup_exec, g, 0);
    cudaGraphDestroy(g);
    if (e != cudaSuccess) return fail(h, PF_ERR_CUDA, std::string("MGS setup graph: ") + cudaGetErrorString(e));
  }
#define MGS_NODE_KERNEL(K, l, ...)                                                  \
  do {                                                                              \
    if (M.lpn[l] == 16) pfb::K<16><<<M.gn[l], pfb::MG_NT, 0, s>>>(__VA_ARGS__); \
    else if (M.lpn[l] == 4) pfb::K<4><<<M.gn[l], pfb::MG_NT, 0, s>>>(__VA_ARGS__); \
    else pfb::K<1><<<M.gn[l], pfb::MG_NT, 0, s>>>(__VA_ARGS__);                     \
  } while (0)
  const int c = nl - 1, top = std::min(A.n_tail, c);
  auto body_kernels = [&](const pfb::MgsArgs& B, bool krylov = true) {
    pfb::k_mgs_fine_resid<<<M.gfr, pfb::MG_NT, 0, s>>>(B);
    for (int l = 1; l < top; ++l) {
      if (M.lpn[l] == 16 && M.fuse && B.L[l].m.n_nodes <= 8192) {
        pfb::k_mgs_sdown<16><<<M.gn[l], pfb::MG_NT, 0, s>>>(B, l);
      } else if (M.lpn[l] == 1 && M.rows && B.L[l].m.n_nodes >= (1 << 20)) {  // large levels: row-table ids (bitwise equal)
        pfb::k_mgs_rrestrict<<<M.gl[l], pfb::MG_NT, 0, s>>>(B, l);
        pfb::k_mgs_rresid<<<M.gl[l], pfb::MG_NT, 0, s>>>(B, l);
      } else {
        MGS_NODE_KERNEL(k_mgs_srestrict, l, B, l);
        MGS_NODE_KERNEL(k_mgs_sresid, l, B, l);
      }
    }
    if (B.n_tail < nl) {
      pfb::k_mgs_tail<<<1, pfb::MG_TAIL_NT, B.ts_bytes, s>>>(B);
    } else {
      MGS_NODE_KERNEL(k_mgs_srestrict, c, B, c);
      if (B.dense) {
        pfb::k_mgs_coarse_dense<<<1, pfb::MG_NT, 0, s>>>(B);
      } else {
        double* bufs[2] = {B.L[c].e, B.L[c].t};
        int cur = (B.nu_c - 1) % 2 == 0 ? 0 : 1;
        pfb::k_mgs_jacobi0<<<M.gn[c], pfb::MG_NT, 0, s>>>(B, c, bufs[cur]);
        for (int k = 1; k < B.nu_c; ++k, cur ^= 1)
          MGS_NODE_KERNEL(k_mgs_ssweep, c, B, c, bufs[cur], bufs[cur ^ 1]);
      }
    }
    for (int l = top - 1; l >= 1; --l) {
      if (M.lpn[l] == 16 && M.fuse) {
        pfb::k_mgs_sup<16><<<M.gn[l], pfb::MG_NT, 0, s>>>(B, l);
      } else if (M.lpn[l] == 1 && M.rows && B.L[l].m.n_nodes >= (1 << 20)) {
        // (the prolongation keeps its 16-byte index table: the row-table version measured
        // 160 us against 131 us at cfg5's level 1)
        MGS_NODE_KERNEL(k_mgs_sprolongate, l, B, l);
        pfb::k_mgs_rsmooth<<<M.gl[l], pfb::MG_NT, 0, s>>>(B, l);
      } else {
        MGS_NODE_KERNEL(k_mgs_sprolongate, l, B, l);
        MGS_NODE_KERNEL(k_mgs_ssmooth, l, B, l);
      }
    }
    pfb::k_mgs_fine_smooth<<<M.gf, pfb::MG_NT, 0, s>>>(B);
    if (!krylov) return;
    pfb::k_mgs_pcg<<<M.gf, pfb::MG_NT, 0, s>>>(B, M.gf);
    pfb::k_mgs_update<<<M.gflat, pfb::MG_NT, 0, s>>>(B, M.gf, M.gf);
  };
  M.body_kernels = 4 + (A.n_tail < nl ? 1 : 1 + (A.dense ? 1 : A.nu_c));
  for (int l = 1; l < top; ++l)
    M.body_kernels += (M.lpn[l] == 16 && M.fuse) ? (A.L[l].m.n_nodes <= 8192 ? 2 : 3) : 4;
  if (h->comm) {  // row strips: the preconditioner only, one V-cycle (pf_mgd.cuh drives the PCG)
    cudaGraph_t g = nullptr;
    A.use_cond = 0;
    PF_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
    body_kernels(A, false);
    PF_CUDA(cudaStreamEndCapture(s, &g));
    cudaError_t e = cudaGraphInstantiate(&M.vcycle_exec, g, 0);
    cudaGraphDestroy(g);
    if (e != cudaSuccess) return fail(h, PF_ERR_CUDA, std::string("MGS V-cycle graph: ") + cudaGetErrorString(e));
    M.vcycle_kernels = M.body_kernels - 2;
    return PF_OK;
  }
  const char* un = getenv("PFB200_MG_UNROLL");
  const int unroll = un ? std::max(0, atoi(un)) : 0;
  if (unroll > 0) {  // profiling only: N unconditional iterations, so ncu sees every kernel
    cudaGraph_t g = nullptr;
    A.use_cond = 0;
    PF_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
    pfb::k_mgs_init<<<M.gflat, pfb::MG_NT, 0, s>>>(A);
    for (int it = 0; it < unroll; ++it) body_kernels(A);
    pfb::k_mgs_finish<<<M.gflat, pfb::MG_NT, 0, s>>>(A);
    PF_CUDA(cudaStreamEndCapture(s, &g));
    cudaError_t e = cudaGraphInstantiate(&M.solve_exec, g, 0);
    cudaGraphDestroy(g);
    if (e != cudaSuccess) return fail(h, PF_ERR_CUDA, std::string("MGS solve graph: ") + cudaGetErrorString(e));
    return PF_OK;
  }
  cudaGraph_t g = nullptr;
  PF_CUDA(cudaGraphCreate(&g, 0));
  PF_CUDA(cudaGraphConditionalHandleCreate(&A.cond, g, 1, cudaGraphCondAssignDefault));
  A.use_cond = 1;
  cudaGraphNode_t n_init = nullptr, n_while = nullptr, n_fin = nullptr;
  {
    cudaGraphNodeParams kp = {};
    kp.type = cudaGraphNodeTypeKernel;
    void* args[] = {&A};
    kp.kernel.func = (void*)pfb::k_mgs_init;
    kp.kernel.gridDim = dim3(M.gflat);
    kp.kernel.blockDim = dim3(pfb::MG_NT);
    kp.kernel.kernelParams = args;
    PF_CUDA(cudaGraphAddNode(&n_init, g, nullptr, 0, &kp));
  }
  cudaGraphNodeParams cp = {};
  cp.type = cudaGraphNodeTypeConditional;
  cp.conditional.handle = A.cond;
  cp.conditional.type = cudaGraphCondTypeWhile;
  cp.conditional.size = 1;
  PF_CUDA(cudaGraphAddNode(&n_while, g, &n_init, 1, &cp));
  cudaGraph_t body = cp.conditional.phGraph_out[0];
  {
    PF_CUDA(cudaStreamBeginCaptureToGraph(s, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
    body_kernels(A);
    cudaGraph_t bb = body;
    PF_CUDA(cudaStreamEndCapture(s, &bb));
  }
  {
    cudaGraphNodeParams kp = {};
    kp.type = cudaGraphNodeTypeKernel;
    void* args[] = {&A};
    kp.kernel.func = (void*)pfb::k_mgs_finish;
    kp.kernel.gridDim = dim3(M.gflat);
    kp.kernel.blockDim = dim3(pfb::MG_NT);
    kp.kernel.kernelParams = args;
    PF_CUDA(cudaGraphAddNode(&n_fin, g, &n_while, 1, &kp));
  }
  cudaError_t e = cudaGraphInstantiate(&M.solve_exec, g, 0);
  cudaGraphDestroy(g);
  if (e != cudaSuccess) return fail(h, PF_ERR_CUDA, std::string("MGS solve graph: ") + cudaGetErrorString(e));
  return PF_OK;
#undef MGS_NODE_KERNEL
}

// Handle creation captures CUDA graphs; a legacy-stream operation (cudaMemcpy / cudaMemset) of
// another thread's concurrent creation would invalidate a capture in progress (several strips
// created by host threads in one process, tests/test_gpu_strips.py).  Creations are serialised,
// except around the strips' solver-path agreement, which needs every rank.
static std::mutex g_create_mu;

static pf_status create_impl(const pf_mesh* mesh, const pf_material* mat, const pf_config* cfg,
                             int device, const pf_strip* strip, pf_handle** out) {
  if (!out || !mesh || !mat || !cfg) return PF_ERR_INVALID;
  std::unique_lock<std::mutex> create_lock(g_create_mu);
  *out = nullptr;
  pf_handle* h = new pf_handle();
  h->device = device;
  h->cfg = *cfg;
  h->mat = *mat;
  pf_status st = validate_mesh(h, mesh);
  if (st != PF_OK) {
    fprintf(stderr, "pf_create: %s\n", h->err.c_str());
    delete h;
    return st;
  }
  auto bail = [&](pf_status s) {
    fprintf(stderr, "pf_create: %s\n", h->err.c_str());
    pf_destroy(h);
    return s;
  };
#define CREATE_CUDA(expr)                                                          \
  do {                                                                             \
    cudaError_t e__ = (expr);                                                      \
    if (e__ != cudaSuccess) {                                                      \
      h->err = std::string("CUDA error: ") + cudaGetErrorString(e__) + " at " #expr; \
      return bail(PF_ERR_CUDA);                                                    \
    }                                                                              \
  } while (0)
  CREATE_CUDA(cudaSetDevice(device));
  CREATE_CUDA(cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking));
  CREATE_CUDA(cudaEventCreate(&h->ev0));
  CREATE_CUDA(cudaEventCreate(&h->ev1));
  CREATE_CUDA(cudaEventCreate(&h->evs0));
  CREATE_CUDA(cudaEventCreate(&h->evs1));
  h->nx = mesh->nx;
  h->ny = mesh->ny;
  h->n_nodes = (int)mesh->n_nodes;
  h->n_elems = (int)mesh->n_elems;
  const int nx = h->nx, ny = h->ny;
  h->h_nlo.assign(mesh->node_lo, mesh->node_lo + ny + 1);
  h->h_nhi.assign(mesh->node_hi, mesh->node_hi + ny + 1);
  h->h_nst.resize(ny + 1);
  for (int j = 0; j <= ny; ++j) h->h_nst[j] = (int)mesh->node_start[j];
  h->h_elo.assign(mesh->elem_lo, mesh->elem_lo + ny);
  h->h_ehi.assign(mesh->elem_hi, mesh->elem_hi + ny);
  h->h_est.resize(ny);
  for (int j = 0; j < ny; ++j) h->h_est[j] = (int)mesh->elem_start[j];
  // active tiles: tiles owning at least one node
  std::vector<int2> tiles;
  const int tiles_x = (nx + 1 + pfb::TX - 1) / pfb::TX, tiles_y = (ny + 1 + pfb::TY - 1) / pfb::TY;
  for (int ty = 0; ty < tiles_y; ++ty)
    for (int tx = 0; tx < tiles_x; ++tx) {
      bool any = false;
      for (int j = ty * pfb::TY; j < std::min((ty + 1) * pfb::TY, ny + 1) && !any; ++j) {
        const int lo = std::max(h->h_nlo[j], tx * pfb::TX), hi = std::min(h->h_nhi[j], (tx + 1) * pfb::TX);
        any = hi > lo;
      }
      if (any) tiles.push_back(make_int2(tx, ty));
    }
  h->n_tiles = (int)tiles.size();
  auto up_int = [&](int** dptr, const std::vector<int>& v) -> cudaError_t {
    cudaError_t e = cudaMalloc((void**)dptr, std::max<size_t>(v.size(), 1) * sizeof(int));
    if (e != cudaSuccess) return e;
    return cudaMemcpy(*dptr, v.data(), v.size() * sizeof(int), cudaMemcpyHostToDevice);
  };
  CREATE_CUDA(up_int(&h->d_nlo, h->h_nlo));
  CREATE_CUDA(up_int(&h->d_nhi, h->h_nhi));
  CREATE_CUDA(up_int(&h->d_nst, h->h_nst));
  CREATE_CUDA(up_int(&h->d_elo, h->h_elo));
  CREATE_CUDA(up_int(&h->d_ehi, h->h_ehi));
  CREATE_CUDA(up_int(&h->d_est, h->h_est));
  CREATE_CUDA(cudaMalloc((void**)&h->d_tiles, tiles.size() * sizeof(int2)));
  CREATE_CUDA(cudaMemcpy(h->d_tiles, tiles.data(), tiles.size() * sizeof(int2), cudaMemcpyHostToDevice));
  {
    std::vector<int4> nrow(ny + 1), erow(std::max(ny, 1));
    for (int j = 0; j <= ny; ++j) nrow[j] = make_int4(h->h_nlo[j], h->h_nhi[j], h->h_nst[j], 0);
    for (int j = 0; j < ny; ++j) erow[j] = make_int4(h->h_elo[j], h->h_ehi[j], h->h_est[j], 0);
    CREATE_CUDA(cudaMalloc((void**)&h->d_nrow, nrow.size() * sizeof(int4)));
    CREATE_CUDA(cudaMalloc((void**)&h->d_erow, erow.size() * sizeof(int4)));
    CREATE_CUDA(cudaMemcpy(h->d_nrow, nrow.data(), nrow.size() * sizeof(int4), cudaMemcpyHostToDevice));
    CREATE_CUDA(cudaMemcpy(h->d_erow, erow.data(), erow.size() * sizeof(int4), cudaMemcpyHostToDevice));
  }
  pfb::DMesh& dm = h->dm;
  dm.nx = nx; dm.ny = ny;
  dm.nlo = h->d_nlo; dm.nhi = h->d_nhi; dm.nst = h->d_nst;
  dm.elo = h->d_elo; dm.ehi = h->d_ehi; dm.est = h->d_est;
  dm.notch_row = mesh->notch_row;
  dm.notch_lo = mesh->notch_row >= 0 ? mesh->notch_lo : 0;
  dm.notch_hi = mesh->notch_row >= 0 ? mesh->notch_hi : 0;
  dm.dup_start = mesh->notch_row >= 0 ? (int)mesh->dup_start : 0;
  dm.n_nodes = h->n_nodes; dm.n_elems = h->n_elems;
  dm.n_tiles = h->n_tiles; dm.tiles = h->d_tiles;
  dm.nrow = h->d_nrow; dm.erow = h->d_erow;
  dm.own_lo = 0; dm.own_hi = h->n_nodes; dm.dup_lo = h->n_nodes;
  dm.cell_lo = 0; dm.cell_hi = h->n_elems;
  if (strip) {
    dm.own_lo = (int)strip->own_lo; dm.own_hi = (int)strip->own_hi; dm.dup_lo = (int)strip->dup_lo;
    dm.cell_lo = (int)strip->cell_lo; dm.cell_hi = (int)strip->cell_hi;
    pfb::HaloSpec sp;
    sp.rank = strip->rank; sp.nranks = strip->nranks;
    sp.send_lo_start = strip->send_lo_start; sp.send_lo_count = strip->send_lo_count;
    sp.recv_lo_start = strip->recv_lo_start; sp.recv_lo_count = strip->recv_lo_count;
    sp.send_hi_start = strip->send_hi_start; sp.send_hi_count = strip->send_hi_count;
    sp.recv_hi_start = strip->recv_hi_start; sp.recv_hi_count = strip->recv_hi_count;
    if (strip->comm_kind == 0) {
      auto* nc = new pfb::NcclComm();
      nc->spec = sp;
      h->comm = nc;
      create_lock.unlock();  // ncclCommInitRank is collective over the ranks
      const std::string e = nc->init(strip->nccl_id);
      create_lock.lock();
      if (!e.empty()) { h->err = e; return bail(PF_ERR_NCCL); }
    } else {
      if (!strip->host_group) { h->err = "host_group is null"; return bail(PF_ERR_INVALID); }
      auto* hc = new pfb::HostComm();
      hc->spec = sp;
      hc->g = static_cast<pfb::HostGroup*>(strip->host_group);
      h->comm = hc;
    }
    CREATE_CUDA(cudaMalloc((void**)&h->d_red, 16 * sizeof(double)));
    CREATE_CUDA(cudaMalloc((void**)&h->gA, pfb::CG_SLOTS * sizeof(double)));
    CREATE_CUDA(cudaMalloc((void**)&h->gB, (pfb::CG_SLOTS + 1) * 2 * sizeof(double)));
  }
  build_consts(h, mesh->hx, mesh->hy);
  h->hx = mesh->hx;
  h->hy = mesh->hy;
  const size_t nn = h->n_nodes, ne = h->n_elems;
  pf_status s2 = PF_OK;
#define CREATE_ALLOC(ptr, n) \
  if ((s2 = dalloc(h, &(ptr), (n))) != PF_OK) return bail(s2)
  CREATE_ALLOC(h->u, 2 * nn);
  CREATE_ALLOC(h->d, nn);
  CREATE_ALLOC(h->dprev, nn);
  CREATE_ALLOC(h->trp, 4 * ne);
  CREATE_ALLOC(h->dev2, 4 * ne);
  CREATE_ALLOC(h->psi, 4 * ne);
  CREATE_ALLOC(h->psimax, 4 * ne);
  CREATE_ALLOC(h->Ru, 2 * nn);
  CREATE_ALLOC(h->ru, 2 * nn);
  CREATE_ALLOC(h->xu, 2 * nn);
  CREATE_ALLOC(h->qu, 2 * nn);
  CREATE_ALLOC(h->p0u, 2 * nn);
  CREATE_ALLOC(h->p1u, 2 * nn);
  {
    // single-reduction momentum PCG (k_cg_sr) by default: per iteration (µs) SR / two-barrier /
    // two-barrier + lazy x: cfg1 9.9 / - / 11.7, cfg2 15.0 / 16.6 / 16.4, cfg4 34.5 / 33.3 /
    // 34.1, cfg3 42.6 / 42.1 / 42.7, cfg5 2290 / 2466 / 2317.  PFB200_SR=0 selects the
    // two-barrier kernel (lazy x for meshes beyond 4x L2).
    h->sr_mom = true;
    const char* srv = getenv("PFB200_SR");
    if (srv) h->sr_mom = std::string(srv) == "1";
    h->sr_mom = h->sr_mom && !strip;  // strips: split-phase kernels
    const char* sre = getenv("PFB200_SR_EVO");
    // Phase-field solves without the SPD probe use the single-reduction PCG (one grid barrier
    // per iteration; cfg2 bench: phase-field time -19%).  Its recurrence stalled once (cfg3's
    // first load step never reached ||r|| < 1e-12 ||b||), so every single-reduction solve runs
    // with an iteration cap and is redone by the two-barrier PCG when it does not converge
    // (evolution() below).  PFB200_SR_EVO=0: two-barrier PCG only.
    h->sr_evo = !(sre && std::string(sre) == "0") && !strip;
    if (h->sr_evo) {
      CREATE_ALLOC(h->r1d, nn);
      CREATE_ALLOC(h->w1d, nn);
      CREATE_ALLOC(h->pcd, nn);
    }
    if (h->sr_mom) {
      CREATE_ALLOC(h->r1u, 2 * nn);
      CREATE_ALLOC(h->w1u, 2 * nn);
      CREATE_ALLOC(h->pcu, 2 * nn);
    }
  }
  CREATE_ALLOC(h->dinvu, 2 * nn);
  CREATE_ALLOC(h->diagu, 2 * nn);
  CREATE_ALLOC(h->flags, ne);
  CREATE_ALLOC(h->umask, 2 * nn);
  CREATE_ALLOC(h->Rd, nn);
  CREATE_ALLOC(h->rd, nn);
  CREATE_ALLOC(h->xd, nn);
  CREATE_ALLOC(h->qd, nn);
  CREATE_ALLOC(h->p0d, nn);
  CREATE_ALLOC(h->p1d, nn);
  CREATE_ALLOC(h->dinvd, nn);
  CREATE_ALLOC(h->diagd, nn);
  CREATE_ALLOC(h->b, 4 * ne);
  CREATE_ALLOC(h->pmask, nn);
  CREATE_ALLOC(h->scratch, 16 * ne);
  {
    const char* w = getenv("PFB200_WARM");
    h->warm = !(w && std::string(w) == "0") && !strip;  // strips: cold starts
    const char* wd = getenv("PFB200_WARM_DEPTH");  // 1..WARM_MAX (A/B tests)
    if (wd) h->warm_depth = std::min(std::max(atoi(wd), 1), pfb::WARM_MAX);
    if (h->warm)
      for (int sl = 0; sl < pf_handle::WARM_SLOTS; ++sl)
        for (int k = 0; k < h->warm_depth; ++k) CREATE_ALLOC(h->warm_buf[sl][k], 2 * nn);
    if (h->warm)
      for (int sl = 0; sl < pf_handle::WARM_SLOTS_D; ++sl)
        for (int k = 0; k < h->warm_depth; ++k) CREATE_ALLOC(h->warm_d[sl][k], nn);
    const char* tr = getenv("PFB200_TRACE");
    h->trace = tr && std::string(tr) == "1";
    const char* mgg = getenv("PFB200_MGS_GATED");
    h->mgs_gated = !(mgg && std::string(mgg) == "0");
  }
  CREATE_CUDA(cudaMemsetAsync(h->umask, 1, 2 * nn, h->stream));
  CREATE_CUDA(cudaMemsetAsync(h->pmask, 1, nn, h->stream));
  int dev_sms = 0, occ = 0, occ_evo = 0, l2 = 0;
  CREATE_CUDA(cudaDeviceGetAttribute(&dev_sms, cudaDevAttrMultiProcessorCount, device));
  CREATE_CUDA(cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, device));
  {  // PFB200_EVO_MARCH=1/0 forces the march form of k_evo_prepare on / off
    const char* em = getenv("PFB200_EVO_MARCH");
    h->evo_march = !strip && (em ? std::string(em) == "1" : h->n_tiles > 65536);
    int oc = 0;
    CREATE_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&oc, pfb::k_evo_prepare_march,
                                                              pfb::MG_NT, 0));
    h->geom_prep = pfb::make_march_geom(nx, ny, std::max(1, oc) * dev_sms * pfb::MG_WARPS);
  }
  {  // both variants of each persistent kernel must be co-resident at the same grid size
    int o1 = 0, o2 = 0;
    CREATE_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o1, pfb::k_cg<true, false>,
                                                              pfb::CG_NT, 0));
    CREATE_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o2, pfb::k_cg<true, true>,
                                                              pfb::CG_NT, 0));
    occ = std::min(o1, o2);
    if (h->sr_mom) {
      h->sr_smem = sizeof(pfb::SrStage<true>) * pfb::SR_SLOTS * (pfb::CG_NT / 32);
      CREATE_CUDA(cudaFuncSetAttribute(pfb::k_cg_sr<true>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)h->sr_smem));
      CREATE_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o2, pfb::k_cg_sr<true>,
                                                                pfb::CG_NT, h->sr_smem));
      occ = std::min(occ, o2);
    }
    CREATE_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o1, pfb::k_cg<false, false>,
                                                              pfb::CG_NT, 0));
    CREATE_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o2, pfb::k_cg<false, true>,
                                                              pfb::CG_NT, 0));
    occ_evo = std::min(o1, o2);
    if (h->sr_evo) {
      h->sr_smem_evo = sizeof(pfb::SrStage<false>) * pfb::SR_SLOTS * (pfb::CG_NT / 32);
      CREATE_CUDA(cudaFuncSetAttribute(pfb::k_cg_sr<false>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)h->sr_smem_evo));
      CREATE_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o2, pfb::k_cg_sr<false>,
                                                                pfb::CG_NT, h->sr_smem_evo));
      occ_evo = std::min(occ_evo, o2);
    }
  }
  h->sm_count = dev_sms;
  h->l2_bytes = l2;
  if (occ < 1 || occ_evo < 1) {
    h->err = "k_cg cannot be resident (occupancy 0)";
    return bail(PF_ERR_CUDA);
  }
  // persistent grids: all resident warps march; unit shape from the resident warp count
  const int wpc = pfb::NT / 32, cwpc = pfb::CG_NT / 32;
  const char* mr = getenv("PFB200_MIN_ROWS");
  const int min_rows = mr ? std::max(1, atoi(mr)) : 4;
  h->geom_mom = pfb::make_march_geom(nx, ny, occ * dev_sms * cwpc, min_rows);
  h->geom_evo = pfb::make_march_geom(nx, ny, occ_evo * dev_sms * cwpc, min_rows);
  h->geom_apply = pfb::make_march_geom(nx, ny, 4 * dev_sms * wpc);
  {  // lazy x update only where one PCG iteration streams far more than L2 holds (measured:
     // 8192^2 -6.5% time per iteration, 1024^2 +2.5% momentum / +10% phase field)
    const double big = 4.0 * (double)l2;
    h->xupd_mom = 168.0 * (double)nn > big;
    h->xupd_evo = 72.0 * (double)nn + 32.0 * (double)ne > big;
    const char* xu = getenv("PFB200_XUPD");  // "0" / "1": force (A/B tests)
    if (xu) h->xupd_mom = h->xupd_evo = std::string(xu) == "1";
  }
  h->cg_grid = std::max(1, std::min(occ * dev_sms, (h->geom_mom.n_units + cwpc - 1) / cwpc));
  h->cg_grid_evo =
      std::max(1, std::min(occ_evo * dev_sms, (h->geom_evo.n_units + cwpc - 1) / cwpc));
  {  // split-phase PCG geometry: phase A one wave of resident CTAs, phase B 4 CTAs per SM
    const char* mode = getenv("PFB200_CG");  // "split": graph-chained phase kernels (A/B tests)
    h->split = mode && std::string(mode) == "split";
    const char* ch = getenv("PFB200_CG_CHUNK");
    if (ch) h->chunk = std::max(1, atoi(ch));
    int oa = 0, oe = 0;
    CREATE_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&oa, pfb::k_cg_a<true>, pfb::NT, 0));
    CREATE_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&oe, pfb::k_cg_a<false>, pfb::NT, 0));
    h->geom_a_mom = pfb::make_march_geom(nx, ny, std::max(oa, 1) * dev_sms * wpc);
    h->geom_a_evo = pfb::make_march_geom(nx, ny, std::max(oe, 1) * dev_sms * wpc);
    h->gridA_mom = (h->geom_a_mom.n_units + wpc - 1) / wpc;
    h->gridA_evo = (h->geom_a_evo.n_units + wpc - 1) / wpc;
    h->gridB = 4 * dev_sms;
    CREATE_CUDA(cudaMalloc((void**)&h->d_ctl, sizeof(pfb::CgCtl)));
    CREATE_CUDA(cudaMallocHost((void**)&h->h_ctl, sizeof(pfb::CgCtl)));
    CREATE_CUDA(cudaMalloc((void**)&h->partA,
                           sizeof(double) * pfb::CG_SLOTS * std::max(h->gridA_mom, h->gridA_evo)));
    CREATE_CUDA(cudaMalloc((void**)&h->partB, sizeof(double) * (pfb::CG_SLOTS + 1) * h->gridB * 2));
  }
  {  // assembled-stencil phase-field PCG (pf_st.cuh) while its rows and vectors (~176 B per
     // node) fit in half of L2; PFB200_ST_EVO=0/1 forces it off/on
    const char* se = getenv("PFB200_ST_EVO");
    h->st_evo = h->sr_evo && !h->comm && !h->split && 176.0 * (double)nn <= 0.5 * (double)l2;
    if (se) h->st_evo = std::string(se) == "1" && h->sr_evo && !h->comm && !h->split;
    if (h->st_evo) {
      int os = 0;
      CREATE_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&os, pfb::k_cg_st, pfb::CG_NT, 0));
      if (os < 1) {
        h->err = "k_cg_st cannot be resident (occupancy 0)";
        return bail(PF_ERR_CUDA);
      }
      const char* so = getenv("PFB200_ST_OCC");  // CTAs per SM (A/B tests)
      if (so) os = std::max(1, std::min(os, atoi(so)));
      h->cg_grid_st = std::max(1, std::min(os * dev_sms, (int)((nn + pfb::CG_NT - 1) / pfb::CG_NT)));
      if ((s2 = st_setup(h)) != PF_OK) return bail(s2);
    }
  }
  const size_t npart =
      std::max<size_t>((size_t)h->n_tiles * 4,
                       (size_t)std::max({h->cg_grid, h->cg_grid_evo, h->cg_grid_st}) *
                           pfb::CG_PART_STRIDE);
  CREATE_ALLOC(h->partials, npart);
  CREATE_CUDA(cudaHostAlloc((void**)&h->h_cgres, sizeof(CgResult), cudaHostAllocMapped));
  CREATE_CUDA(cudaHostGetDevicePointer((void**)&h->d_cgres, h->h_cgres, 0));
  CREATE_CUDA(cudaHostAlloc((void**)&h->h_scal, 16 * sizeof(double), cudaHostAllocMapped));
  CREATE_CUDA(cudaHostGetDevicePointer((void**)&h->d_scal, h->h_scal, 0));
  {  // geometric-multigrid PCG for the momentum solves (single GPU; PFB200_MG=0: Jacobi PCG)
    const char* mgv = getenv("PFB200_MG");
    // row strips: strip-local V-cycles as a block-Jacobi preconditioner (pf_mgd.cuh;
    // PFB200_DIST_MG=0: the split-phase Jacobi PCG)
    const char* dmg = getenv("PFB200_DIST_MG");
    const bool dist_mg = !(dmg && std::string(dmg) == "0");
    const bool want = !(mgv && std::string(mgv) == "0") && (!strip || dist_mg);
    if (strip) {  // level 0 of the strip hierarchies: the first owned node row onwards
      for (int j = 0; j <= ny; ++j)
        if (h->h_nst[j] == (int)strip->own_lo) { h->mgd_row0 = j; break; }
    }
    if (want) {
      int om = 0, o2 = 0;
      CREATE_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&om, pfb::k_mg_fine_smooth, pfb::MG_NT, 0));
      CREATE_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o2, pfb::k_mg_pcg, pfb::MG_NT, 0));
      om = std::min(om, o2);
      CREATE_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o2, pfb::k_mg_fine_resid, pfb::MG_NT, 0));
      om = std::min(om, o2);
      if (om >= 1) {
        pf_status ms = mg_setup(h, h->mgu, 0, om * dev_sms * pfb::MG_WARPS);
        if (ms != PF_OK) return bail(ms);
        // phase-field multigrid (solves without the SPD probe) where Jacobi PCG iteration
        // counts get large: deep hierarchies on big meshes (PFB200_MG_EVO=1/0: force on/off)
        // PFB200_MG_EVO: "1" / "scalar" the native scalar hierarchy (pf_mgs.cuh), "packed" the
        // round-1 two-component packing (pf_mg.cuh phys 1, A/B comparisons), "0" off
        const char* me = getenv("PFB200_MG_EVO");
        const bool evo_auto = h->mgu.on && h->mgu.A.n_levels >= 5 && h->n_nodes >= 500000;
        const std::string mev = me ? std::string(me) : std::string(evo_auto ? "scalar" : "0");
        if (mev == "packed" && h->mgu.on) {
          pf_status es = mg_setup(h, h->mgd, 1, om * dev_sms * pfb::MG_WARPS);
          if (es != PF_OK) return bail(es);
        } else if ((mev == "1" || mev == "scalar") && h->mgu.on) {
          int os = 0, o3 = 0;
          CREATE_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&os, pfb::k_mgs_fine_smooth, pfb::MG_NT, 0));
          CREATE_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o3, pfb::k_mgs_pcg, pfb::MG_NT, 0));
          os = std::min(os, o3);
          CREATE_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o3, pfb::k_mgs_fine_resid, pfb::MG_NT, 0));
          os = std::max(1, std::min(os, o3));
          pf_status es = mgs_setup(h, h->mgs, os * dev_sms * pfb::MG_WARPS);
          if (es != PF_OK) return bail(es);
        }
        if (strip) {  // every strip must take the same solver path (collectives): agree
          double* d_flag = nullptr;
          CREATE_CUDA(cudaMalloc((void**)&d_flag, 2 * sizeof(double)));
          const double miss[2] = {h->mgu.on ? 0.0 : 1.0, h->mgs.on ? 0.0 : 1.0};
          CREATE_CUDA(cudaMemcpy(d_flag, miss, sizeof miss, cudaMemcpyHostToDevice));
          create_lock.unlock();  // every rank must reach the all-reduce
          const std::string ce = h->comm->allreduce(d_flag, 2, h->stream);
          create_lock.lock();
          double tot[2] = {0.0, 0.0};
          cudaMemcpyAsync(tot, d_flag, sizeof tot, cudaMemcpyDeviceToHost, h->stream);
          cudaStreamSynchronize(h->stream);
          cudaFree(d_flag);
          if (!ce.empty()) { h->err = ce; return bail(PF_ERR_NCCL); }
          if (tot[0] > 0.0) h->mgu.on = false;  // some strip's rows do not coarsen: Jacobi PCG
          if (tot[1] > 0.0) h->mgs.on = false;
        }
        if (strip && (h->mgu.on || h->mgs.on)) {  // the strip PCG's scalars, partials, marches
          CREATE_CUDA(cudaMalloc((void**)&h->d_mgd, 8 * sizeof(double)));
          CREATE_CUDA(cudaMemset(h->d_mgd, 0, 8 * sizeof(double)));
          CREATE_CUDA(cudaMallocHost((void**)&h->h_mgd, 8 * sizeof(double)));
          int ou = 0, od = 0;
          CREATE_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ou, pfb::k_mgd_dir_mom, pfb::MG_NT, 0));
          CREATE_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&od, pfb::k_mgd_dir_pf, pfb::MG_NT, 0));
          h->mgd_geom_u = pfb::make_march_geom(nx, ny, std::max(1, ou) * dev_sms * pfb::MG_WARPS);
          h->mgd_geom_d = pfb::make_march_geom(nx, ny, std::max(1, od) * dev_sms * pfb::MG_WARPS);
          h->mgd_gdir_u = (h->mgd_geom_u.n_units + pfb::MG_WARPS - 1) / pfb::MG_WARPS;
          h->mgd_gdir_d = (h->mgd_geom_d.n_units + pfb::MG_WARPS - 1) / pfb::MG_WARPS;
          h->mgd_gflat = 2 * dev_sms;
          const int np = std::max({h->mgd_gflat, h->mgd_gdir_u, h->mgd_gdir_d});
          CREATE_CUDA(cudaMalloc((void**)&h->mgd_part, np * sizeof(double)));
        }
        const char* mw = getenv("PFB200_MG_WARM");  // "0": MG solves start cold (x0 = 0)
        if (h->mgu.on && mw && std::string(mw) == "0") h->warm = false;
        const char* ru = getenv("PFB200_MG_REUSE");
        h->mgu.reuse = !(ru && std::string(ru) == "0");
        // the phase-field tangent changes strongly between Newton iterations (cfg5: 10-18
        // iterations on a fresh hierarchy, 50-74 on the previous one): rebuild every solve
        h->mgd.reuse = ru && std::string(ru) == "1";
      }
    }
  }
  CREATE_CUDA(cudaStreamSynchronize(h->stream));
  *out = h;
  return PF_OK;
#undef CREATE_ALLOC
#undef CREATE_CUDA
}

extern "C" pf_status pf_create(const pf_mesh* mesh, const pf_material* mat, const pf_config* cfg,
                               int device, pf_handle** out) {
  return create_impl(mesh, mat, cfg, device, nullptr, out);
}

extern "C" pf_status pf_create_strip(const pf_mesh* local_mesh, const pf_material* mat,
                                     const pf_config* cfg, int device, const pf_strip* strip,
                                     pf_handle** out) {
  if (!strip || strip->nranks < 1 || strip->rank < 0 || strip->rank >= strip->nranks)
    return PF_ERR_INVALID;
  return create_impl(local_mesh, mat, cfg, device, strip, out);
}

extern "C" pf_status pf_nccl_unique_id(unsigned char out[128]) {
  pfb::NcclApi& api = pfb::NcclApi::get();
  const std::string e = api.load();
  if (!e.empty()) {
    fprintf(stderr, "pf_nccl_unique_id: %s\n", e.c_str());
    return PF_ERR_NCCL;
  }
  ncclUniqueId id;
  if (api.GetUniqueId(&id) != ncclSuccess) return PF_ERR_NCCL;
  std::memcpy(out, &id, sizeof(id) < 128 ? sizeof(id) : 128);
  return PF_OK;
}

extern "C" pf_status pf_host_group_create(int32_t nranks, void** out) {
  if (nranks < 1 || !out) return PF_ERR_INVALID;
  *out = new pfb::HostGroup(nranks);
  return PF_OK;
}

extern "C" void pf_host_group_destroy(void* group) { delete static_cast<pfb::HostGroup*>(group); }

// ------------------------------------------------------------------------------------------
// state transfer.  Host arrays are ordinary (pageable) caller memory: large transfers go through
// one pinned staging buffer, the host-side copy split over a few threads (the driver's pageable
// path is a single-threaded staged copy; fresh output arrays also fault their pages in there).
struct Xfer {
  double* host;
  double* dev;
  size_t n;
};

// bytes-balanced parallel memcpy over a list of (dst, src, bytes) segments
static void par_copy(const std::vector<std::array<size_t, 3>>& seg) {
  size_t total = 0;
  for (const auto& sg : seg) total += sg[2];
  const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
  const size_t nt = std::min<size_t>({(size_t)8, (size_t)hw, std::max<size_t>(1, total >> 22)});
  auto run = [&](size_t lo, size_t hi) {  // global byte range [lo, hi)
    size_t base = 0;
    for (const auto& sg : seg) {
      const size_t a = std::max(lo, base), b = std::min(hi, base + sg[2]);
      if (a < b)
        std::memcpy(reinterpret_cast<char*>(sg[0]) + (a - base),
                    reinterpret_cast<const char*>(sg[1]) + (a - base), b - a);
      base += sg[2];
    }
  };
  if (nt <= 1) return run(0, total);
  std::vector<std::thread> th;
  const size_t step = (total + nt - 1) / nt;
  for (size_t t = 1; t < nt; ++t) th.emplace_back(run, t * step, std::min(total, (t + 1) * step));
  run(0, std::min(total, step));
  for (auto& t : th) t.join();
}

static pf_status ensure_stage(pf_handle* h, size_t n) {
  if (n <= h->stage_cap) return PF_OK;
  if (h->stage) cudaFreeHost(h->stage);
  h->stage = nullptr;
  h->stage_cap = 0;
  PF_CUDA(cudaHostAlloc((void**)&h->stage, n * sizeof(double), cudaHostAllocDefault));
  h->stage_cap = n;
  return PF_OK;
}

static constexpr size_t STAGE_MIN = 1 << 19;  // doubles (4 MB): below, plain pageable copies

// page-locked host memory (pf_host_alloc, cudaHostAlloc / cudaHostRegister): DMA directly
static bool host_pinned(const void* p) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

static pf_status transfer(pf_handle* h, const std::vector<Xfer>& items0, bool to_device) {
  // pinned host buffers go straight to / from the device; the rest through the staging buffer
  std::vector<Xfer> items;
  for (const auto& it : items0) {
    if (!it.host) continue;
    if (host_pinned(it.host)) {
      PF_CUDA(cudaMemcpyAsync(to_device ? (void*)it.dev : (void*)it.host,
                              to_device ? (const void*)it.host : (const void*)it.dev,
                              it.n * sizeof(double),
                              to_device ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToHost,
                              h->stream));
    } else {
      items.push_back(it);
    }
  }
  size_t total = 0;
  for (const auto& it : items)
    if (it.host) total += it.n;
  if (total < STAGE_MIN) {
    for (const auto& it : items)
      if (it.host)
        PF_CUDA(cudaMemcpyAsync(to_device ? (void*)it.dev : (void*)it.host,
                                to_device ? (const void*)it.host : (const void*)it.dev,
                                it.n * sizeof(double),
                                to_device ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToHost,
                                h->stream));
    PF_CUDA(cudaStreamSynchronize(h->stream));
    return PF_OK;
  }
  PF_TRY(ensure_stage(h, total));
  std::vector<std::array<size_t, 3>> seg;
  size_t off = 0;
  for (const auto& it : items) {
    if (!it.host) continue;
    double* st = h->stage + off;
    if (to_device) seg.push_back({(size_t)st, (size_t)it.host, it.n * sizeof(double)});
    else seg.push_back({(size_t)it.host, (size_t)st, it.n * sizeof(double)});
    off += it.n;
  }
  if (to_device) par_copy(seg);
  off = 0;
  for (const auto& it : items) {
    if (!it.host) continue;
    PF_CUDA(cudaMemcpyAsync(to_device ? (void*)it.dev : (void*)(h->stage + off),
                            to_device ? (const void*)(h->stage + off) : (const void*)it.dev,
                            it.n * sizeof(double),
                            to_device ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToHost,
                            h->stream));
    off += it.n;
  }
  PF_CUDA(cudaStreamSynchronize(h->stream));
  if (!to_device) par_copy(seg);
  return PF_OK;
}

static pf_status h2d(pf_handle* h, double* dst, const double* src, size_t n) {
  return transfer(h, {{const_cast<double*>(src), dst, n}}, true);
}
static pf_status d2h(pf_handle* h, double* dst, const double* src, size_t n) {
  return transfer(h, {{dst, const_cast<double*>(src), n}}, false);
}

extern "C" pf_status pf_set_state(pf_handle* h, const double* u, const double* d,
                                  const double* d_prev, const double* trp, const double* dev2,
                                  const double* psi, const double* psimax) {
  if (!h) return PF_ERR_INVALID;
  PF_CUDA(cudaSetDevice(h->device));
  const size_t nn = h->n_nodes, ng = 4 * (size_t)h->n_elems;
  auto c = [](const double* p) { return const_cast<double*>(p); };
  return transfer(h,
                  {{c(u), h->u, 2 * nn}, {c(d), h->d, nn}, {c(d_prev), h->dprev, nn},
                   {c(trp), h->trp, ng}, {c(dev2), h->dev2, ng}, {c(psi), h->psi, ng},
                   {c(psimax), h->psimax, ng}},
                  true);
}

// Device-side state construction: the zero state of SolverState.zeros (schemes.py:80-87) plus
// d = d_prev = 1 at the pre-crack nodes (configs.precrack_nodes), without host arrays.
extern "C" pf_status pf_init_state(pf_handle* h, const double* segments, int64_t n_segments,
                                   double radius, double x_last, double y_last) {
  if (!h) return PF_ERR_INVALID;
  PF_CUDA(cudaSetDevice(h->device));
  if (h->comm) return fail(h, PF_ERR_INVALID, "pf_init_state: single-GPU handles only");
  if (n_segments < 0 || (n_segments > 0 && !segments))
    return fail(h, PF_ERR_INVALID, "pf_init_state: bad segment list");
  const size_t nn = h->n_nodes, ng = 4 * (size_t)h->n_elems;
  for (auto pr : {std::make_pair(h->u, 2 * nn), std::make_pair(h->d, nn),
                  std::make_pair(h->dprev, nn), std::make_pair(h->trp, ng),
                  std::make_pair(h->dev2, ng), std::make_pair(h->psi, ng),
                  std::make_pair(h->psimax, ng)})
    PF_CUDA(cudaMemsetAsync(pr.first, 0, pr.second * sizeof(double), h->stream));
  if (n_segments > 0) {
    double4* dseg = nullptr;
    PF_CUDA(cudaMallocAsync((void**)&dseg, (size_t)n_segments * sizeof(double4), h->stream));
    PF_CUDA(cudaMemcpyAsync(dseg, segments, (size_t)n_segments * sizeof(double4),
                            cudaMemcpyHostToDevice, h->stream));
    pfb::k_precrack<<<8 * h->sm_count, 256, 0, h->stream>>>(h->dm, h->hx, h->hy, x_last, y_last,
                                                          dseg, (int)n_segments, radius, h->d,
                                                          h->dprev);
    PF_TRY(launched(h));
    PF_CUDA(cudaFreeAsync(dseg, h->stream));
  }
  PF_CUDA(cudaStreamSynchronize(h->stream));
  return PF_OK;
}

extern "C" pf_status pf_get_state(pf_handle* h, double* u, double* d, double* d_prev,
                                  double* trp, double* dev2, double* psi, double* psimax) {
  if (!h) return PF_ERR_INVALID;
  PF_CUDA(cudaSetDevice(h->device));
  const size_t nn = h->n_nodes, ng = 4 * (size_t)h->n_elems;
  return transfer(h,
                  {{u, h->u, 2 * nn}, {d, h->d, nn}, {d_prev, h->dprev, nn}, {trp, h->trp, ng},
                   {dev2, h->dev2, ng}, {psi, h->psi, ng}, {psimax, h->psimax, ng}},
                  false);
}

static dim3 cell_grid(const pf_handle* h) { return dim3((h->nx + 127) / 128, h->ny); }

static pfb::GpArgs gp_args(pf_handle* h) {
  pfb::GpArgs g{};
  g.m = h->dm;
  g.C = h->C;
  g.u = reinterpret_cast<const double2*>(h->u);
  g.d = h->d;
  g.trp = h->trp;
  g.dev2 = h->dev2;
  g.psi = h->psi;
  g.psimax = h->psimax;
  return g;
}

// page-locked host buffers for state outputs (direct DMA in pf_get_state / pf_get_gp_strain)
extern "C" pf_status pf_host_alloc(int64_t bytes, void** out) {
  if (!out || bytes <= 0) return PF_ERR_INVALID;
  *out = nullptr;
  if (cudaHostAlloc(out, (size_t)bytes, cudaHostAllocPortable) != cudaSuccess) {
    cudaGetLastError();
    return PF_ERR_CUDA;
  }
  return PF_OK;
}
extern "C" void pf_host_free(void* p) {
  if (p) cudaFreeHost(p);
}

extern "C" pf_status pf_get_gp_strain(pf_handle* h, double* strain, double* tr_eps) {
  if (!h) return PF_ERR_INVALID;
  PF_CUDA(cudaSetDevice(h->device));
  const size_t ne = h->n_elems;
  double* tr_dev = h->scratch;  // tr first (4 ne), then strain needs 16 ne: do two passes
  pfb::GpArgs g = gp_args(h);
  g.trp = nullptr; g.dev2 = nullptr; g.psi = nullptr;
  if (tr_eps) {
    g.tr = tr_dev;
    pfb::k_refresh_gp<<<cell_grid(h), 128, 0, h->stream>>>(g);
    PF_TRY(launched(h));
    PF_TRY(d2h(h, tr_eps, tr_dev, 4 * ne));
  }
  if (strain) {
    g.tr = nullptr;
    g.strain = h->scratch;
    pfb::k_refresh_gp<<<cell_grid(h), 128, 0, h->stream>>>(g);
    PF_TRY(launched(h));
    PF_TRY(d2h(h, strain, h->scratch, 16 * ne));
  }
  return PF_OK;
}

// interp_nodal (assembly.py:148-150) of a host nodal field: [n_nodes] -> [n_elems*4]
extern "C" pf_status pf_interp_nodal(pf_handle* h, const double* field, double* out) {
  if (!h) return PF_ERR_INVALID;
  if (!field || !out) return fail(h, PF_ERR_INVALID, "pf_interp_nodal: null array");
  PF_CUDA(cudaSetDevice(h->device));
  const size_t nn = h->n_nodes, ne = h->n_elems;
  double* fd = h->scratch;                        // scratch holds 16 n_elems doubles
  double* od = h->scratch + ((nn + 1) & ~size_t(1));  // >= nn, 16-byte aligned
  if (((nn + 1) & ~size_t(1)) + 4 * ne > 16 * ne)
    return fail(h, PF_ERR_INVALID, "pf_interp_nodal: mesh too small for the scratch buffer");
  PF_TRY(h2d(h, fd, field, nn));
  pfb::k_interp_nodal<<<cell_grid(h), 128, 0, h->stream>>>(gp_args(h), fd, od);
  PF_TRY(launched(h));
  return d2h(h, out, od, 4 * ne);
}

// ------------------------------------------------------------------------------------------
// masks
static pf_status set_umask(pf_handle* h, const std::vector<int64_t>& cons) {
  if (cons == h->cons_key) return PF_OK;
  const size_t n = 2 * (size_t)h->n_nodes;
  std::vector<uint8_t> m(n, 1);
  for (int64_t k : cons) {
    if (k < 0 || (size_t)k >= n) return fail(h, PF_ERR_INDEX, "constrained node outside the system");
    m[k] = 0;
  }
  PF_CUDA(cudaMemcpyAsync(h->umask, m.data(), n, cudaMemcpyHostToDevice, h->stream));
  PF_CUDA(cudaStreamSynchronize(h->stream));
  h->mgu.built = false;  // the Galerkin levels are masked at the Dirichlet dofs
  h->cons_key = cons;
  h->umask_all_free = cons.empty();
  return PF_OK;
}

static pf_status set_pmask(pf_handle* h, const int64_t* pins, int64_t n_pins) {
  std::vector<int64_t> key(pins, pins + (pins ? n_pins : 0));
  if (key == h->pins_key) return PF_OK;
  const size_t n = h->n_nodes;
  std::vector<uint8_t> m(n, 1);
  for (int64_t k : key) {
    if (k < 0 || (size_t)k >= n) return fail(h, PF_ERR_INDEX, "constrained node outside the system");
    m[k] = 0;
  }
  PF_CUDA(cudaMemcpyAsync(h->pmask, m.data(), n, cudaMemcpyHostToDevice, h->stream));
  PF_CUDA(cudaStreamSynchronize(h->stream));
  h->n_pinned = (int64_t)std::count(m.begin(), m.end(), (uint8_t)0);
  h->mgd.built = false;  // the phase-field Galerkin levels are masked at the pinned nodes
  h->pins_key = key;
  h->pmask_all_free = key.empty();
  return PF_OK;
}

static pf_status ensure_idx(pf_handle* h, size_t n) {
  if (n <= h->d_idx_cap) return PF_OK;
  if (h->d_idx) cudaFree(h->d_idx);
  h->d_idx_cap = std::max<size_t>(n, 1024);
  PF_CUDA(cudaMalloc((void**)&h->d_idx, h->d_idx_cap * sizeof(long long)));
  return PF_OK;
}

// ------------------------------------------------------------------------------------------
// kernel launch helpers
static pf_status launch_mom_prepare(pf_handle* h, int full) {
  pfb::MomPrepArgs a{};
  a.m = h->dm;
  a.C = h->C;
  a.u = reinterpret_cast<const double2*>(h->u);
  a.d = h->d;
  a.umask = reinterpret_cast<const uchar2*>(h->umask);
  a.R = reinterpret_cast<double2*>(h->Ru);
  a.r = reinterpret_cast<double2*>(h->ru);
  a.x = reinterpret_cast<double2*>(h->xu);
  a.dinv = reinterpret_cast<double2*>(h->dinvu);
  a.flags = h->flags;
  a.diag = reinterpret_cast<double2*>(h->diagu);
  a.partials = h->partials;
  a.full = full;
  pfb::k_mom_prepare<<<h->n_tiles, pfb::NT, 0, h->stream>>>(a);
  h->parts_n = h->n_tiles;  // (a prepare kernel without a finalize may have left its own count)
  return launched(h);
}

static pf_status launch_evo_prepare(pf_handle* h, int full, int extra_scheme) {
  pfb::EvoPrepArgs a{};
  a.m = h->dm;
  a.C = h->C;
  a.d = h->d;
  a.dprev = h->dprev;
  a.psi = h->psi;
  a.trp = h->trp;
  a.dev2 = h->dev2;
  a.psimax = h->psimax;
  a.pmask = h->pmask;
  a.R = h->Rd;
  a.r = h->rd;
  a.x = h->xd;
  a.dinv = h->dinvd;
  a.b = h->b;
  a.diag = h->diagd;
  a.partials = h->partials;
  a.full = full;
  a.extra_scheme = extra_scheme;
  if (h->evo_march) {  // big meshes: one warp march (pf_mgs.cuh k_evo_prepare_march)
    const int grid = (h->geom_prep.n_units + pfb::MG_WARPS - 1) / pfb::MG_WARPS;
    pfb::k_evo_prepare_march<<<grid, pfb::MG_NT, 0, h->stream>>>(a, h->geom_prep);
    h->parts_n = grid;
    return launched(h);
  }
  pfb::k_evo_prepare<<<h->n_tiles, pfb::NT, 0, h->stream>>>(a);
  h->parts_n = h->n_tiles;
  return launched(h);
}

static pf_status comm_check(pf_handle* h, const std::string& e) {
  if (e.empty()) return PF_OK;
  return fail(h, PF_ERR_NCCL, e);
}

// sums nv partial streams of n_tiles CTAs into h_scal[0..nv) (all-reduced over the strips) and
// waits for them
static pf_status finalize(pf_handle* h, int nv) {
  // one CTA sums the per-tile partials in a fixed order; 1024 threads on the big meshes (the
  // 256-thread order is kept below 2^16 tiles: the small cases' norms stay bit-identical)
  const int np = h->parts_n > 0 ? h->parts_n : h->n_tiles;
  const int nt = np > 65536 ? 1024 : 256;
  h->parts_n = 0;
  if (!h->comm) {
    pfb::k_finalize<<<1, nt, 0, h->stream>>>(h->partials, np, nv, h->d_scal);
    PF_TRY(launched(h));
    PF_CUDA(cudaStreamSynchronize(h->stream));
    return PF_OK;
  }
  pfb::k_finalize<<<1, nt, 0, h->stream>>>(h->partials, np, nv, h->d_red);
  PF_TRY(launched(h));
  PF_TRY(comm_check(h, h->comm->allreduce(h->d_red, nv, h->stream)));
  PF_CUDA(cudaMemcpyAsync(h->h_scal, h->d_red, nv * sizeof(double), cudaMemcpyDeviceToHost,
                          h->stream));
  PF_CUDA(cudaStreamSynchronize(h->stream));
  return PF_OK;
}

static pf_status halo(pf_handle* h, double* vec, int comps) {
  if (!h->comm) return PF_OK;
  return comm_check(h, h->comm->halo(vec, comps, h->stream));
}

static pf_status axpy(pf_handle* h, double* y, const double* x, long long n) {
  pfb::k_axpy<<<(unsigned)((n + 255) / 256), 256, 0, h->stream>>>(y, x, n);
  return launched(h);
}

static size_t cg_smem(const pf_handle* h, bool mom) {  // dynamic smem of the chosen PCG kernel
  return mom ? (h->sr_mom ? h->sr_smem : 0) : (h->sr_evo_now ? h->sr_smem_evo : 0);
}

static const void* cg_kernel(pf_handle* h, bool mom) {
  if (mom && h->sr_mom) return (const void*)pfb::k_cg_sr<true>;
  if (!mom && h->st_evo_now) return (const void*)pfb::k_cg_st;
  if (!mom && h->sr_evo_now) return (const void*)pfb::k_cg_sr<false>;
  if (mom) return h->xupd_mom ? (const void*)pfb::k_cg<true, true> : (const void*)pfb::k_cg<true, false>;
  return h->xupd_evo ? (const void*)pfb::k_cg<false, true> : (const void*)pfb::k_cg<false, false>;
}

static pfb::CgArgs cg_args(pf_handle* h, bool mom) {
  pfb::CgArgs a{};
  a.m = h->dm;
  a.C = h->C;
  a.vec2 = mom ? 1 : 0;
  a.ndof = mom ? 2LL * h->n_nodes : (long long)h->n_nodes;
  a.g = mom ? h->geom_mom : h->geom_evo;
  a.d = h->d;
  a.flags = h->flags;
  a.b = h->b;
  a.x = mom ? h->xu : h->xd;
  a.r = mom ? h->ru : h->rd;
  a.q = mom ? h->qu : h->qd;
  a.p0 = mom ? h->p0u : h->p0d;
  a.p1 = mom ? h->p1u : h->p1d;
  a.r1 = mom ? h->r1u : h->r1d;
  a.w1 = mom ? h->w1u : h->w1d;
  a.pc = mom ? h->pcu : h->pcd;
  a.dinv = mom ? h->dinvu : h->dinvd;
  a.partials = h->partials;
  a.result = h->d_cgres;
  a.rtol = h->cfg.cg_rtol;
  a.maxiter = (long long)h->cfg.cg_maxiter_factor * a.ndof;  // 20 * matrix.shape[0]
  return a;
}

static pf_status cg_account(pf_handle* h, bool mom, long long iters, float ms) {
  const double nfree_u = 2.0 * h->n_nodes - (double)h->cons_key.size();
  const double nfree_d = (double)h->n_nodes - (double)h->n_pinned;
  if (mom) {
    h->acc.cg_iters_u += iters;
    h->acc.cg_dofiters_u += (double)iters * nfree_u;
    h->acc.kernel_ms_u += ms;
    h->acc.cg_launches_u += 1;
  } else {
    h->acc.cg_iters_d += iters;
    h->acc.cg_dofiters_d += (double)iters * nfree_d;
    h->acc.kernel_ms_d += ms;
    h->acc.cg_launches_d += 1;
  }
  return PF_OK;
}

static pf_status cg_status(pf_handle* h, int status, long long iters) {
  if (status == pfb::CG_MAXITER)
    return fail(h, PF_ERR_SINGULAR, "cg failed to converge (info=" + std::to_string(iters) + ")");
  if (status == pfb::CG_NAN) return fail(h, PF_ERR_SINGULAR, "cg produced a non-finite residual");
  return PF_OK;
}

// one persistent PCG solve (single cooperative launch)
static pf_status run_cg_persistent(pf_handle* h, bool mom, double* target, bool probe,
                                   int* status, long long* iters, double* const* guess,
                                   int n_guess, long long maxiter_cap = 0) {
  pfb::CgArgs a = cg_args(h, mom);
  if (maxiter_cap > 0) a.maxiter = std::min(a.maxiter, maxiter_cap);
  a.target = target;
  a.probe = probe ? 1 : 0;
  for (int k = 0; k < n_guess && k < pfb::WARM_MAX; ++k) a.guess[k] = guess[k];
  a.n_guess = guess ? std::min(n_guess, pfb::WARM_MAX) : 0;
  void* args[] = {&a, &h->st};  // (k_cg_st only reads the second)
  const void* fn = cg_kernel(h, mom);
  const int grid = mom ? h->cg_grid : (h->st_evo_now ? h->cg_grid_st : h->cg_grid_evo);
  PF_CUDA(cudaEventRecord(h->ev0, h->stream));
  PF_CUDA(cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(pfb::CG_NT), args,
                                      cg_smem(h, mom), h->stream));
  PF_TRY(launched(h));
  PF_CUDA(cudaEventRecord(h->ev1, h->stream));
  PF_CUDA(cudaStreamSynchronize(h->stream));
  float ms = 0.f;
  PF_CUDA(cudaEventElapsedTime(&ms, h->ev0, h->ev1));
  *status = h->h_cgres->status;
  *iters = h->h_cgres->iters;
  cg_account(h, mom, *iters, ms);
  return cg_status(h, *status, *iters);
}

static pfb::SplitArgs split_args(pf_handle* h, bool mom, bool probe) {
  pfb::SplitArgs s{};
  s.c = cg_args(h, mom);
  s.c.g = mom ? h->geom_a_mom : h->geom_a_evo;
  s.c.probe = probe ? 1 : 0;
  s.ctl = h->d_ctl;
  s.partA = h->partA;
  s.partB = h->partB;
  s.gridA = mom ? h->gridA_mom : h->gridA_evo;
  s.gridB = h->gridB;
  return s;
}

// a CUDA graph of `chunk` iterations (phase A, phase B) + the base advance, cached per handle
static pf_status chunk_graph(pf_handle* h, bool mom, bool probe, cudaGraphExec_t* out) {
  cudaGraphExec_t& g = h->graphs[mom ? 1 : 0][probe ? 1 : 0];
  if (!g) {
    pfb::SplitArgs s = split_args(h, mom, probe);
    cudaGraph_t graph;
    PF_CUDA(cudaStreamBeginCapture(h->stream, cudaStreamCaptureModeThreadLocal));
    for (int kl = 0; kl < h->chunk; ++kl) {
      if (mom) {
        pfb::k_cg_a<true><<<s.gridA, pfb::NT, 0, h->stream>>>(s, kl);
        pfb::k_cg_b<true><<<s.gridB, pfb::NT, 0, h->stream>>>(s, kl);
      } else {
        pfb::k_cg_a<false><<<s.gridA, pfb::NT, 0, h->stream>>>(s, kl);
        pfb::k_cg_b<false><<<s.gridB, pfb::NT, 0, h->stream>>>(s, kl);
      }
    }
    pfb::k_cg_advance<<<1, 1, 0, h->stream>>>(h->d_ctl, h->chunk);
    PF_CUDA(cudaStreamEndCapture(h->stream, &graph));
    PF_CUDA(cudaGraphInstantiate(&g, graph, 0));
    PF_CUDA(cudaGraphDestroy(graph));
  }
  *out = g;
  return PF_OK;
}

static pf_status run_cg_split(pf_handle* h, bool mom, double* target, bool probe, int* status,
                              long long* iters) {
  pfb::SplitArgs s = split_args(h, mom, probe);
  cudaGraphExec_t g;
  PF_TRY(chunk_graph(h, mom, probe, &g));
  PF_CUDA(cudaEventRecord(h->ev0, h->stream));
  PF_CUDA(cudaMemsetAsync(h->d_ctl, 0, sizeof(pfb::CgCtl), h->stream));
  if (mom) pfb::k_cg_init<true><<<s.gridB, pfb::NT, 0, h->stream>>>(s);
  else pfb::k_cg_init<false><<<s.gridB, pfb::NT, 0, h->stream>>>(s);
  PF_TRY(launched(h));
  for (;;) {
    PF_CUDA(cudaGraphLaunch(g, h->stream));
    h->acc.launches += 2 * h->chunk + 1;
    PF_CUDA(cudaMemcpyAsync(h->h_ctl, h->d_ctl, sizeof(pfb::CgCtl), cudaMemcpyDeviceToHost,
                            h->stream));
    PF_CUDA(cudaStreamSynchronize(h->stream));
    if (h->h_ctl->done) break;
  }
  *status = h->h_ctl->status;
  *iters = h->h_ctl->iters;
  if (*status == pfb::CG_CONVERGED && target) {
    const long long n = s.c.ndof;
    pfb::k_cg_finish<<<4 * h->sm_count, 256, 0, h->stream>>>(target, s.c.x, n);
    PF_TRY(launched(h));
  }
  PF_CUDA(cudaEventRecord(h->ev1, h->stream));
  PF_CUDA(cudaStreamSynchronize(h->stream));
  float ms = 0.f;
  PF_CUDA(cudaEventElapsedTime(&ms, h->ev0, h->ev1));
  cg_account(h, mom, *iters, ms);
  return cg_status(h, *status, *iters);
}

// split-phase PCG with all-reduces and halo exchanges between the phases (row strips).
// Every rank takes identical decisions because every decision uses all-reduced scalars.
static pf_status run_cg_dist(pf_handle* h, bool mom, double* target, bool probe, int* status,
                             long long* iters) {
  pfb::SplitArgs s = split_args(h, mom, probe);
  s.gA = h->gA;
  s.gB = h->gB;
  const int comps = mom ? 2 : 1;
  PF_CUDA(cudaEventRecord(h->ev0, h->stream));
  PF_CUDA(cudaMemsetAsync(h->d_ctl, 0, sizeof(pfb::CgCtl), h->stream));
  if (mom) pfb::k_cg_init<true><<<s.gridB, pfb::NT, 0, h->stream>>>(s);
  else pfb::k_cg_init<false><<<s.gridB, pfb::NT, 0, h->stream>>>(s);
  PF_TRY(launched(h));
  double* gb0 = h->gB + 2 * pfb::CG_SLOTS;
  pfb::k_finalize<<<1, 256, 0, h->stream>>>(h->partB + (size_t)pfb::CG_SLOTS * s.gridB * 2,
                                            s.gridB, 2, gb0);
  PF_TRY(launched(h));
  PF_TRY(comm_check(h, h->comm->allreduce(gb0, 2, h->stream)));
  // one iteration k = k0 + kl (kl < chunk, chunk % 6 == 0 so slot and parity depend on kl only)
  auto iteration = [&](int kl) -> pf_status {
    const int sl = kl % pfb::CG_SLOTS;
    if (mom) pfb::k_cg_a<true><<<s.gridA, pfb::NT, 0, h->stream>>>(s, kl);
    else pfb::k_cg_a<false><<<s.gridA, pfb::NT, 0, h->stream>>>(s, kl);
    PF_TRY(launched(h));
    pfb::k_finalize<<<1, 256, 0, h->stream>>>(h->partA + (size_t)sl * s.gridA, s.gridA, 1,
                                              h->gA + sl);
    PF_TRY(launched(h));
    PF_TRY(comm_check(h, h->comm->allreduce(h->gA + sl, 1, h->stream)));
    if (mom) pfb::k_cg_b<true><<<s.gridB, pfb::NT, 0, h->stream>>>(s, kl);
    else pfb::k_cg_b<false><<<s.gridB, pfb::NT, 0, h->stream>>>(s, kl);
    PF_TRY(launched(h));
    pfb::k_finalize<<<1, 256, 0, h->stream>>>(h->partB + (size_t)sl * s.gridB * 2, s.gridB, 2,
                                              h->gB + 2 * sl);
    PF_TRY(launched(h));
    PF_TRY(comm_check(h, h->comm->allreduce(h->gB + 2 * sl, 2, h->stream)));
    PF_TRY(halo(h, s.c.r, comps));
    PF_TRY(halo(h, (kl & 1) ? s.c.p1 : s.c.p0, comps));
    return PF_OK;
  };
  const int chunk = std::max(6, (h->chunk / 6) * 6);
  cudaGraphExec_t* gexec = &h->dgraphs[mom ? 1 : 0][probe ? 1 : 0];
  if (h->comm->capturable() && !*gexec) {  // record the chunk once: kernels + NCCL
    cudaGraph_t graph;
    PF_CUDA(cudaStreamBeginCapture(h->stream, cudaStreamCaptureModeThreadLocal));
    pf_status st = PF_OK;
    for (int kl = 0; kl < chunk && st == PF_OK; ++kl) st = iteration(kl);
    pfb::k_cg_advance<<<1, 1, 0, h->stream>>>(h->d_ctl, chunk);
    cudaError_t ce = cudaStreamEndCapture(h->stream, &graph);
    if (st != PF_OK) return st;
    PF_CUDA(ce);
    PF_CUDA(cudaGraphInstantiate(gexec, graph, 0));
    PF_CUDA(cudaGraphDestroy(graph));
  }
  for (;;) {
    if (h->comm->capturable()) {
      PF_CUDA(cudaGraphLaunch(*gexec, h->stream));
      h->acc.launches += 5 * chunk + 1;
    } else {
      for (int kl = 0; kl < chunk; ++kl) PF_TRY(iteration(kl));
      pfb::k_cg_advance<<<1, 1, 0, h->stream>>>(h->d_ctl, chunk);
      PF_TRY(launched(h));
    }
    PF_CUDA(cudaMemcpyAsync(h->h_ctl, h->d_ctl, sizeof(pfb::CgCtl), cudaMemcpyDeviceToHost,
                            h->stream));
    PF_CUDA(cudaStreamSynchronize(h->stream));
    if (h->h_ctl->done) break;
  }
  *status = h->h_ctl->status;
  *iters = h->h_ctl->iters;
  if (*status == pfb::CG_CONVERGED && target) PF_TRY(axpy(h, target, s.c.x, s.c.ndof));
  PF_CUDA(cudaEventRecord(h->ev1, h->stream));
  PF_CUDA(cudaStreamSynchronize(h->stream));
  float ms = 0.f;
  PF_CUDA(cudaEventElapsedTime(&ms, h->ev0, h->ev1));
  cg_account(h, mom, *iters, ms);
  return cg_status(h, *status, *iters);
}


// one MG-PCG solve: setup graph (hierarchy at the current tangent), then the solve graph whose
// PCG loop is a device-side WHILE node; the host waits once, at the end
static pf_status run_mg(pf_handle* h, MgInst& M, double* target, int* status, long long* iters,
                        int setup_only = 0, long long maxiter = -1, double rtol = -1.0,
                        bool check = true, bool force_setup = false,
                        double* const* guess = nullptr, int n_guess = 0) {
  M.in->n_guess = std::min(n_guess, pfb::MG_WARM);
  for (int k = 0; k < pfb::MG_WARM; ++k) M.in->guess[k] = k < M.in->n_guess ? guess[k] : nullptr;
  M.in->rtol = rtol >= 0.0 ? rtol : h->cfg.cg_rtol;
  M.in->maxiter = maxiter > 0 ? maxiter
                                  : (long long)h->cfg.cg_maxiter_factor * 2LL * h->n_nodes;
  M.in->target = target;
  const bool rebuild = force_setup || setup_only || !M.reuse || !M.built ||
                       M.age >= M.max_age ||
                       M.last_iters > (M.ref_iters * 5) / 4 + 2;
  // a reused hierarchy gets an iteration budget: past it the solve reports CG_MAXITER and the
  // caller redoes it on a fresh hierarchy (crack steps change the tangent quickly)
  if (!rebuild && maxiter <= 0 && M.reuse_cap)
    M.in->maxiter = std::min(M.in->maxiter, std::max(50LL, 3 * M.ref_iters + 20));
  PF_CUDA(cudaEventRecord(h->ev0, h->stream));
  PF_CUDA(cudaMemcpyAsync((void*)M.A.in, M.in, sizeof(pfb::MgIn), cudaMemcpyHostToDevice,
                          h->stream));
  if (rebuild) {
    PF_CUDA(cudaGraphLaunch(M.setup_exec, h->stream));
    PF_TRY(launched(h));
    M.setups += 1;
  }
  if (!setup_only) {
    PF_CUDA(cudaGraphLaunch(M.solve_exec, h->stream));
    PF_TRY(launched(h));
  }
  PF_CUDA(cudaEventRecord(h->ev1, h->stream));
  PF_CUDA(cudaStreamSynchronize(h->stream));
  float ms = 0.f;
  PF_CUDA(cudaEventElapsedTime(&ms, h->ev0, h->ev1));
  if (rebuild) {
    M.built = true;
    M.age = 0;
  }
  if (setup_only) return PF_OK;
  *status = h->h_cgres->status;
  *iters = h->h_cgres->iters;
  if (rebuild) M.ref_iters = *iters;
  M.last_iters = *iters;
  // kernels executed inside the graphs (each graph launch counted one by launched())
  h->acc.launches += (rebuild ? M.setup_kernels - 1 : 0) +
                     (setup_only ? 0 : pfb::MG_WARM + 1 + (int)(*iters) * M.body_kernels);
  if (h->trace)
    fprintf(stderr, "[pfb200] mg solve: %lld iterations, %.3f ms%s\n", *iters, ms,
            rebuild ? " (hierarchy rebuilt)" : "");
  if (M.A.tclk) {
    long long c[32] = {};
    cudaMemcpy(c, M.A.tclk, sizeof c, cudaMemcpyDeviceToHost);
    fprintf(stderr, "[pfb200] tail phases (cycles):");
    for (int k = 1; k < 32 && c[k]; ++k) fprintf(stderr, " %lld", c[k] - c[k - 1]);
    fprintf(stderr, "\n");
  }
  M.age += 1;
  if (!check) return PF_OK;
  cg_account(h, M.A.phys == 0, *iters, ms);
  return cg_status(h, *status, *iters);
}

// one scalar phase-field MG-PCG solve on (rd, dinvd, b): fresh hierarchy, then the solve graph
// (device-side WHILE); the solution lands in xd, rd is consumed
static pf_status run_mgs(pf_handle* h, MgsInst& M, int* status, long long* iters,
                         long long maxiter = -1, double rtol = -1.0, bool check = true,
                         bool safe = false, bool probe = false) {
  M.in->n_guess = 0;
  M.in->probe = probe ? 1 : 0;
  M.in->rtol = rtol >= 0.0 ? rtol : h->cfg.cg_rtol;
  M.in->maxiter = maxiter > 0 ? maxiter : (long long)h->cfg.cg_maxiter_factor * h->n_nodes;
  M.in->target = nullptr;
  PF_CUDA(cudaEventRecord(h->ev0, h->stream));
  PF_CUDA(cudaMemcpyAsync((void*)M.A.in, M.in, sizeof(pfb::MgIn), cudaMemcpyHostToDevice,
                          h->stream));
  PF_CUDA(cudaGraphLaunch(safe ? M.setup_safe_exec : M.setup_exec, h->stream));
  PF_TRY(launched(h));
  PF_CUDA(cudaGraphLaunch(M.solve_exec, h->stream));
  PF_TRY(launched(h));
  PF_CUDA(cudaEventRecord(h->ev1, h->stream));
  PF_CUDA(cudaStreamSynchronize(h->stream));
  float ms = 0.f;
  PF_CUDA(cudaEventElapsedTime(&ms, h->ev0, h->ev1));
  M.setups += 1;
  *status = h->h_cgres->status;
  *iters = h->h_cgres->iters;
  // kernels inside the two graphs (each graph launch was counted once by launched()):
  // setup kernels, init, iterations x body, finish
  h->acc.launches += (safe ? M.setup_kernels_safe : M.setup_kernels) - 1 + 2 +
                     (int)(*iters) * M.body_kernels - 1;
  if (h->trace)
    fprintf(stderr, "[pfb200] scalar phase-field mg solve: %lld iterations, %.3f ms\n", *iters, ms);
  if (!check) return PF_OK;
  cg_account(h, false, *iters, ms);
  return cg_status(h, *status, *iters);
}

// The multigrid PCG on a row strip (pf_mgd.cuh): local V-cycles as a block-Jacobi
// preconditioner, the Krylov recurrence with NCCL (or host-group) all-reduces and halo rows;
// x ends up in xu / xd (ghost rows to be refreshed by the caller's halo exchange).
static pf_status run_mgd(pf_handle* h, bool mom, int* status, long long* iters) {
  const int comps = mom ? 2 : 1;
  cudaStream_t s = h->stream;
  double* g = h->d_mgd;
  double* r = mom ? h->ru : h->rd;
  double* x = mom ? h->xu : h->xd;
  double* q = mom ? h->qu : h->qd;
  double* p0 = mom ? h->p0u : h->p0d;
  double* p1 = mom ? h->p1u : h->p1d;
  const double* dinv = mom ? h->dinvu : h->dinvd;
  double* vdinv = mom ? h->mgu.A.L[0].dinv : h->mgs.A.L[0].dinv;
  double* z = mom ? h->mgu.A.z : h->mgs.A.z;
  const int gfl = h->mgd_gflat;
  // the interface row (first owned node row of ranks > 0): point Jacobi in the preconditioner
  const int if_lo = h->mgd_row0 > 0 ? h->h_nst[h->mgd_row0] : 0;
  const int if_hi = h->mgd_row0 > 0 ? if_lo + (h->h_nhi[h->mgd_row0] - h->h_nlo[h->mgd_row0]) : 0;
  PF_CUDA(cudaEventRecord(h->ev0, s));
  pfb::k_mgd_mask<<<gfl, 256, 0, s>>>(vdinv, dinv, comps, h->dm, if_lo, if_hi);
  if (mom) {
    PF_CUDA(cudaGraphLaunch(h->mgu.setup_exec, s));
    h->acc.launches += h->mgu.setup_kernels;
    h->mgu.setups += 1;
  } else {
    MgsInst& M = h->mgs;  // strips: the safe (MG_POW-step) hierarchy
    PF_CUDA(cudaGraphLaunch(M.setup_safe_exec, s));
    h->acc.launches += M.setup_kernels_safe;
    M.setups += 1;
  }
  pfb::k_mgd_init<<<gfl, pfb::MG_NT, 0, s>>>(x, r, comps, h->dm, h->mgd_part);
  pfb::k_finalize<<<1, 256, 0, s>>>(h->mgd_part, gfl, 1, g + pfb::MGD_RR);
  h->acc.launches += 3;
  PF_TRY(comm_check(h, h->comm->allreduce(g + pfb::MGD_RR, 1, s)));
  PF_CUDA(cudaMemcpyAsync(h->h_mgd, g + pfb::MGD_RR, sizeof(double), cudaMemcpyDeviceToHost, s));
  PF_CUDA(cudaStreamSynchronize(s));
  const double bnorm = std::sqrt(h->h_mgd[0]);
  const double atol = h->cfg.cg_rtol * bnorm;
  const long long maxiter = (long long)h->cfg.cg_maxiter_factor * comps * h->n_nodes *
                            std::max(1, h->comm->spec.nranks);
  long long k = 0;
  int st = pfb::CG_CONVERGED;
  if (bnorm > 0.0 && !(bnorm < atol)) {
    const pfb::MarchGeom& gd = mom ? h->mgd_geom_u : h->mgd_geom_d;
    const int gdir = mom ? h->mgd_gdir_u : h->mgd_gdir_d;
    for (k = 0;; ++k) {
      PF_CUDA(cudaGraphLaunch(mom ? h->mgu.vcycle_exec : h->mgs.vcycle_exec, s));  // z = M^-1 r
      if (if_hi > if_lo)
        pfb::k_mgd_iface<<<std::max(1, (comps * (if_hi - if_lo) + 255) / 256), 256, 0, s>>>(
            z, r, dinv, comps, if_lo, if_hi);
      if (k > 0) pfb::k_mgd_shift<<<1, 1, 0, s>>>(g);
      pfb::k_mgd_dot<<<gfl, pfb::MG_NT, 0, s>>>(r, z, comps, h->dm, h->mgd_part);
      pfb::k_finalize<<<1, 256, 0, s>>>(h->mgd_part, gfl, 1, g + pfb::MGD_RZ);
      PF_TRY(comm_check(h, h->comm->allreduce(g + pfb::MGD_RZ, 1, s)));
      PF_TRY(halo(h, z, comps));
      const double* pold = (k & 1) ? p0 : p1;
      double* pnew = (k & 1) ? p1 : p0;
      if (mom)
        pfb::k_mgd_dir_mom<<<gdir, pfb::MG_NT, 0, s>>>(h->mgu.A, h->dm, gd, dinv, g, k == 0, pold,
                                                        pnew, h->mgd_part);
      else
        pfb::k_mgd_dir_pf<<<gdir, pfb::MG_NT, 0, s>>>(h->mgs.A, h->dm, gd, dinv, g, k == 0, pold,
                                                       pnew, h->mgd_part);
      pfb::k_finalize<<<1, 256, 0, s>>>(h->mgd_part, gdir, 1, g + pfb::MGD_PQ);
      PF_TRY(comm_check(h, h->comm->allreduce(g + pfb::MGD_PQ, 1, s)));
      pfb::k_mgd_update<<<gfl, pfb::MG_NT, 0, s>>>(x, r, pnew, q, comps, h->dm, g, h->mgd_part);
      pfb::k_finalize<<<1, 256, 0, s>>>(h->mgd_part, gfl, 1, g + pfb::MGD_RR);
      PF_TRY(comm_check(h, h->comm->allreduce(g + pfb::MGD_RR, 1, s)));
      PF_CUDA(cudaMemcpyAsync(h->h_mgd, g + pfb::MGD_RR, sizeof(double), cudaMemcpyDeviceToHost, s));
      PF_CUDA(cudaStreamSynchronize(s));
      PF_CUDA(cudaGetLastError());
      h->acc.launches += (mom ? h->mgu.vcycle_kernels : h->mgs.vcycle_kernels) + 7 + (k > 0) +
                         (if_hi > if_lo);
      const double rn = std::sqrt(h->h_mgd[0]);
      if (rn < atol) { ++k; st = pfb::CG_CONVERGED; break; }
      if (!(rn == rn)) { ++k; st = pfb::CG_NAN; break; }
      if (k + 1 >= maxiter) { ++k; st = pfb::CG_MAXITER; break; }
    }
  }
  PF_CUDA(cudaEventRecord(h->ev1, s));
  PF_CUDA(cudaStreamSynchronize(s));
  float ms = 0.f;
  PF_CUDA(cudaEventElapsedTime(&ms, h->ev0, h->ev1));
  *status = st;
  *iters = k;
  if (h->trace)
    fprintf(stderr, "[pfb200] strip mg-pcg (%s): %lld iterations, %.3f ms\n",
            mom ? "momentum" : "phase field", k, ms);
  cg_account(h, mom, k, ms);
  return cg_status(h, st, k);
}

static pf_status run_cg(pf_handle* h, bool mom, double* target, bool probe, int* status,
                        long long* iters, double* const* guess = nullptr, int n_guess = 0) {
  if (h->comm && !probe && (mom ? h->mgu.on : h->mgs.on)) {
    if (target) return fail(h, PF_ERR_INVALID, "strip multigrid PCG: no target update");
    return run_mgd(h, mom, status, iters);
  }
  if (mom && h->mgu.on && !probe)
    return run_mg(h, h->mgu, target, status, iters, 0, -1, -1.0, true, false, guess, n_guess);
  if (h->comm) return run_cg_dist(h, mom, target, probe, status, iters);
  return h->split ? run_cg_split(h, mom, target, probe, status, iters)
                  : run_cg_persistent(h, mom, target, probe, status, iters, guess, n_guess);
}

// ------------------------------------------------------------------------------------------
// solve_momentum (schemes.py:192-239)
struct BcView {
  const int64_t* dofs;
  const int64_t* offsets;
  const double* incs;
  int n;
};

static pf_status momentum(pf_handle* h, const BcView& bc, bool apply_inc, double* r0,
                          int* n_nr_out, double* last_ratio, int pass) {
  // kinematic increments (schemes.py:207-209): u[dofs] += inc for unique dofs of each pair
  std::vector<int64_t> cons;
  for (int k = 0; k < bc.n; ++k) {
    std::vector<int64_t> dofs(bc.dofs + bc.offsets[k], bc.dofs + bc.offsets[k + 1]);
    for (int64_t v : dofs)
      if (v < 0 || v >= 2LL * h->n_nodes)
        return fail(h, PF_ERR_INDEX, "index out of bounds in boundary-condition dofs");
    std::sort(dofs.begin(), dofs.end());
    dofs.erase(std::unique(dofs.begin(), dofs.end()), dofs.end());
    cons.insert(cons.end(), dofs.begin(), dofs.end());
    if (apply_inc && bc.incs[k] != 0.0 && !dofs.empty()) {
      PF_TRY(ensure_idx(h, dofs.size()));
      PF_CUDA(cudaMemcpyAsync(h->d_idx, dofs.data(), dofs.size() * sizeof(long long),
                              cudaMemcpyHostToDevice, h->stream));
      const long long n = (long long)dofs.size();
      pfb::k_add_inc<<<(unsigned)((n + 255) / 256), 256, 0, h->stream>>>(h->u, h->d_idx, n,
                                                                          bc.incs[k]);
      PF_TRY(launched(h));
      PF_CUDA(cudaStreamSynchronize(h->stream));  // d_idx is reused by the next pair
    }
  }
  std::sort(cons.begin(), cons.end());
  cons.erase(std::unique(cons.begin(), cons.end()), cons.end());
  PF_TRY(set_umask(h, cons));
  const pf_config& cfg = h->cfg;
  int n_nr = 0;
  double rnorm = 0.0;
  for (int it = 0; it <= cfg.max_nr; ++it) {
    PF_TRY(launch_mom_prepare(h, 1));
    PF_TRY(finalize(h, 1));
    rnorm = std::sqrt(h->h_scal[0]);
    if (std::isnan(*r0)) *r0 = rnorm;
    if (rnorm <= std::max(cfg.tol_nr * *r0, cfg.res_floor)) break;
    if (it == cfg.max_nr) {
      char buf[256];
      snprintf(buf, sizeof buf,
               "momentum Newton loop did not converge in %d iterations (relative residual %.3e)",
               cfg.max_nr, rnorm / std::max(*r0, cfg.res_floor));
      return fail(h, PF_ERR_CONV_MOMENTUM, buf);
    }
    int status;
    long long iters;
    if (h->comm) {  // ghost rows of r and D^-1 from their owners; u ghosts refreshed below
      PF_TRY(halo(h, h->ru, 2));
      PF_TRY(halo(h, h->dinvu, 2));
      PF_TRY(run_cg(h, true, nullptr, false, &status, &iters));
      PF_TRY(halo(h, h->xu, 2));
      PF_TRY(axpy(h, h->u, h->xu, 2LL * h->n_nodes));
    } else {
      // warm start of the first Newton step from the previous solve of the same kind (the
      // load-increment pass or a staggered pass); later Newton corrections start from zero
      const int ws = std::min(std::max(pass, 0), pf_handle::WARM_SLOTS - 1);
      double* guess[pfb::WARM_MAX] = {};
      const int ng = (h->warm && n_nr == 0) ? h->warm_n[ws] : 0;
      for (int k = 0; k < ng; ++k) guess[k] = h->warm_buf[ws][k];
      pf_status cst;
      if (h->mgu.on) {
        h->mgu.reuse_cap = true;
        cst = run_cg(h, true, h->u, false, &status, &iters, guess, ng);
        h->mgu.reuse_cap = false;
        if (cst == PF_ERR_SINGULAR && status == pfb::CG_MAXITER && h->mgu.age > 1) {
          // the reused hierarchy was too stale: u is untouched (target is updated only on
          // convergence); rebuild and redo the solve from the same Newton residual
          if (h->trace)
            fprintf(stderr, "[pfb200] mg solve over budget (%lld iterations): rebuild, redo\n", iters);
          PF_TRY(launch_mom_prepare(h, 1));
          PF_TRY(finalize(h, 1));
          h->mgu.built = false;
          cst = run_cg(h, true, h->u, false, &status, &iters, guess, ng);
        }
      } else {
        cst = run_cg(h, true, h->u, false, &status, &iters, guess, ng);
      }
      PF_TRY(cst);
      if (h->trace)
        fprintf(stderr, "[pfb200] momentum pass %d newton %d warm %d iters %lld\n", pass, n_nr,
                ng, iters);
      if (h->warm && n_nr == 0) {  // the solution joins the difference table
        // (the multigrid solves read only the first MG_WARM entries: deeper ones are not kept)
        const int depth = h->mgu.on ? std::min(h->warm_depth, pfb::MG_WARM) : h->warm_depth;
        pfb::WarmTable t{};
        for (int k = 0; k < depth; ++k) t.d[k] = h->warm_buf[ws][k];
        const long long n = 2LL * h->n_nodes;
        pfb::k_warm_push<<<16 * h->sm_count, 256, 0, h->stream>>>(t, h->warm_n[ws], depth, h->xu, n);
        PF_TRY(launched(h));
        h->warm_n[ws] = std::min(h->warm_n[ws] + 1, depth);
      }
    }
    n_nr += 1;
  }
  // refresh_gp_from_displacement (assembly.py:260-269)
  pfb::GpArgs g = gp_args(h);
  pfb::k_refresh_gp<<<cell_grid(h), 128, 0, h->stream>>>(g);
  PF_TRY(launched(h));
  *n_nr_out = n_nr;
  *last_ratio = rnorm / std::max(*r0, cfg.res_floor);
  return PF_OK;
}

// solve_evolution (schemes.py:242-313)
static pf_status evolution(pf_handle* h, int scheme, double* r0, int* n_nr_out, int* fallbacks,
                           int pass = 0) {
  const pf_config& cfg = h->cfg;
  int n_nr = 0;
  for (int it = 0; it <= cfg.max_nr; ++it) {
    const int extra = (it == 0 && scheme != PF_ST) ? scheme : 0;
    PF_TRY(launch_evo_prepare(h, 1, extra));
    PF_TRY(finalize(h, 3));
    const double rnorm = std::sqrt(h->h_scal[0]);
    const bool gated = extra != 0 && h->h_scal[1] > 0.0;
    const bool nonpos_diag = h->h_scal[2] > 0.0;
    if (std::isnan(*r0)) *r0 = rnorm;
    if (rnorm <= std::max(cfg.tol_nr * *r0, cfg.res_floor)) break;
    if (it == cfg.max_nr) {
      char buf[256];
      snprintf(buf, sizeof buf,
               "evolution Newton loop did not converge in %d iterations (relative residual %.3e)",
               cfg.max_nr, rnorm / std::max(*r0, cfg.res_floor));
      return fail(h, PF_ERR_CONV_EVOLUTION, buf);
    }
    int status = pfb::CG_CONVERGED;
    long long iters = 0;
    if (h->comm) {
      PF_TRY(halo(h, h->rd, 1));
      PF_TRY(halo(h, h->dinvd, 1));
    }
    if (gated) {
      // SPD predicate for K_dd + K~ (replaces check_spd, linsolve.py:58-77): a non-positive
      // diagonal, or non-positive curvature p.Ap inside PCG, means "not positive definite"
      bool fallback = nonpos_diag;
      const bool mgs_gated = h->mgs.on && !h->comm && h->mgs_gated;
      if (!fallback) {
        bool decided = false;
        if (mgs_gated) {
          // the probe inside the scalar multigrid PCG (k_mgs_update): p.Ap <= 0 => not positive
          // definite; converged => the Jacobi PCG's verdict "no non-positive curvature met".
          // Anything else (iteration budget, a non-finite residual from a hierarchy built on an
          // indefinite matrix) decides nothing: the Jacobi-PCG probe below redoes the solve.
          MgsInst& M = h->mgs;
          const long long budget = std::max(100LL, 4 * M.last_iters);
          const pf_status ms = run_mgs(h, M, &status, &iters, budget, -1.0, true, false, true);
          if (ms != PF_OK && !(ms == PF_ERR_SINGULAR &&
                               (status == pfb::CG_MAXITER || status == pfb::CG_NAN)))
            return ms;
          if (ms == PF_OK && status == pfb::CG_INDEFINITE) {
            fallback = decided = true;
          } else if (ms == PF_OK) {
            M.last_iters = iters;
            decided = true;
          } else {
            if (h->trace)
              fprintf(stderr, "[pfb200] gated phase-field mg solve undecided (status %d, %lld "
                              "iterations): Jacobi-PCG probe\n", status, iters);
            M.redos += 1;
            PF_TRY(launch_evo_prepare(h, 1, extra));  // the solve consumed the right-hand side
          }
        }
        if (!decided) {
          PF_TRY(run_cg(h, false, nullptr, true, &status, &iters));
          fallback = status == pfb::CG_INDEFINITE;
        }
      }
      if (fallback) {  // plain tangent for this staggered iteration (schemes.py:293-301)
        PF_TRY(launch_evo_prepare(h, 1, 0));
        if (h->comm) {
          PF_TRY(halo(h, h->rd, 1));
          PF_TRY(halo(h, h->dinvd, 1));
        }
        bool solved = false;
        if (mgs_gated) {
          MgsInst& M = h->mgs;
          const long long budget = std::max(100LL, 4 * M.last_iters);
          const pf_status ms = run_mgs(h, M, &status, &iters, budget);
          if (ms != PF_OK && !(ms == PF_ERR_SINGULAR &&
                               (status == pfb::CG_MAXITER || status == pfb::CG_NAN)))
            return ms;
          solved = ms == PF_OK;
          if (solved) M.last_iters = iters;
          else PF_TRY(launch_evo_prepare(h, 1, 0));
        }
        if (!solved) PF_TRY(run_cg(h, false, nullptr, false, &status, &iters));
        *fallbacks += 1;
      }
      PF_TRY(halo(h, h->xd, 1));
      // one-time half-step energy update from this increment (schemes.py:303-310)
      pfb::GpArgs g = gp_args(h);
      g.dd = h->xd;
      g.scheme = scheme;
      pfb::k_update_energy<<<cell_grid(h), 128, 0, h->stream>>>(g);
      PF_TRY(launched(h));
      const long long n = h->n_nodes;
      pfb::k_axpy<<<(unsigned)((n + 255) / 256), 256, 0, h->stream>>>(h->d, h->xd, n);
      PF_TRY(launched(h));
    } else if (h->comm) {
      PF_TRY(run_cg(h, false, nullptr, false, &status, &iters));
      PF_TRY(halo(h, h->xd, 1));
      PF_TRY(axpy(h, h->d, h->xd, h->n_nodes));
    } else {
      // warm start of the first Newton step from the previous solves of the same staggered
      // pass (no SPD probe here: the system is K_dd without K~)
      const int ws = std::min(std::max(pass - 1, 0), pf_handle::WARM_SLOTS_D - 1);
      const bool use_warm = h->warm && n_nr == 0 && pass > 0;
      double* guess[pfb::WARM_MAX] = {};
      const int ng = use_warm ? h->warm_nd[ws] : 0;
      for (int k = 0; k < ng; ++k) guess[k] = h->warm_d[ws][k];
      bool done = false;
      if (h->mgs.on && !h->comm) {
        // native scalar multigrid PCG (pf_mgs.cuh) on the phase-field system in place, on the
        // fast hierarchy with an iteration budget; past it, the solve is redone on the safe one
        MgsInst& M = h->mgs;
        const long long budget = std::max(100LL, 4 * M.last_iters);
        pf_status ms = run_mgs(h, M, &status, &iters, budget);
        if (ms == PF_ERR_SINGULAR && (status == pfb::CG_MAXITER || status == pfb::CG_NAN)) {
          if (h->trace)
            fprintf(stderr, "[pfb200] phase-field mg solve over budget (%lld iterations): safe "
                            "hierarchy, redo\n", iters);
          M.redos += 1;
          PF_TRY(launch_evo_prepare(h, 1, 0));  // the solve consumed the right-hand side
          ms = run_mgs(h, M, &status, &iters, -1, -1.0, true, true);
        }
        PF_TRY(ms);
        M.last_iters = iters;
        PF_TRY(axpy(h, h->d, h->xd, h->n_nodes));
        done = true;
      }
      if (!done && h->mgd.on && !h->comm) {
        // multigrid PCG on the packed two-component layout (pf_mg.cuh, phys 1)
        const long long n = h->n_nodes;
        const unsigned gb = (unsigned)std::min<long long>((n + 255) / 256, 8LL * h->sm_count);
        auto attempt = [&](bool cap) -> pf_status {
          pfb::k_mg_pack2<<<gb, 256, 0, h->stream>>>(h->mgd.A.r, h->rd, n);
          pfb::k_mg_pack2<<<gb, 256, 0, h->stream>>>(h->mgd.A.L[0].dinv, h->dinvd, n);
          PF_TRY(launched(h));
          h->mgd.reuse_cap = cap;
          const pf_status st2 = run_mg(h, h->mgd, nullptr, &status, &iters);
          h->mgd.reuse_cap = false;
          return st2;
        };
        pf_status est = attempt(true);
        if (est == PF_ERR_SINGULAR && status == pfb::CG_MAXITER && h->mgd.age > 1) {
          if (h->trace)
            fprintf(stderr, "[pfb200] phase-field mg solve over budget (%lld iterations): "
                            "rebuild, redo\n", iters);
          PF_TRY(launch_evo_prepare(h, 1, 0));
          h->mgd.built = false;
          est = attempt(false);
        }
        PF_TRY(est);
        pfb::k_mg_unpack_add<<<gb, 256, 0, h->stream>>>(h->xd, h->d, h->mgd.A.x, n);
        PF_TRY(launched(h));
        done = true;
      }
      if (!done && h->sr_evo && !h->comm && !h->split) {
        // single-reduction PCG with an iteration cap (4x the last converged phase-field solve);
        // d is updated only after it converged
        const long long cap = std::max(300LL, 4 * h->evo_last_iters);
        if (h->st_evo) {  // assemble this solve's rows (b and D^-1 from launch_evo_prepare)
          pfb::k_evo_stencil<<<(unsigned)((h->n_nodes + 255) / 256), 256, 0, h->stream>>>(
              h->st, h->C, h->b, h->dinvd);
          PF_TRY(launched(h));
        }
        h->sr_evo_now = !h->st_evo;
        h->st_evo_now = h->st_evo;
        const pf_status sst = run_cg_persistent(h, false, nullptr, false, &status, &iters, guess,
                                                ng, cap);
        h->sr_evo_now = h->st_evo_now = false;
        if (sst == PF_OK) {
          PF_TRY(axpy(h, h->d, h->xd, h->n_nodes));
          done = true;
        } else if (sst != PF_ERR_SINGULAR) {
          return sst;
        } else {  // stalled: redo this solve from scratch with the two-barrier PCG
          if (h->trace)
            fprintf(stderr, "[pfb200] single-reduction phase-field PCG stalled after %lld "
                            "iterations: two-barrier PCG\n", iters);
          PF_TRY(launch_evo_prepare(h, 1, 0));
        }
      }
      if (!done) PF_TRY(run_cg(h, false, h->d, false, &status, &iters, guess, ng));
      h->evo_last_iters = iters;
      if (use_warm) {
        pfb::WarmTable t{};
        for (int k = 0; k < h->warm_depth; ++k) t.d[k] = h->warm_d[ws][k];
        pfb::k_warm_push<<<16 * h->sm_count, 256, 0, h->stream>>>(t, h->warm_nd[ws], h->warm_depth,
                                                              h->xd, (long long)h->n_nodes);
        PF_TRY(launched(h));
        h->warm_nd[ws] = std::min(h->warm_nd[ws] + 1, h->warm_depth);
      }
    }
    if (h->trace)
      fprintf(stderr, "[pfb200] evolution newton %d gated %d iters %lld\n", n_nr, (int)gated,
              iters);
    n_nr += 1;
  }
  *n_nr_out = n_nr;
  return PF_OK;
}

static pf_status evo_norm(pf_handle* h, double* out) {
  PF_TRY(launch_evo_prepare(h, 0, 0));
  PF_TRY(finalize(h, 3));
  *out = std::sqrt(h->h_scal[0]);
  return PF_OK;
}

static pf_status commit(pf_handle* h) {
  const long long ngp = 4LL * h->n_elems, nn = h->n_nodes;
  const long long n = std::max(ngp, nn);
  pfb::k_commit<<<(unsigned)((n + 255) / 256), 256, 0, h->stream>>>(h->psimax, h->psi, ngp,
                                                                    h->dprev, h->d, nn);
  return launched(h);
}

// ------------------------------------------------------------------------------------------
extern "C" pf_status pf_staggered_step(pf_handle* h, int scheme, const int64_t* bc_dofs,
                                       const int64_t* bc_offsets, const double* bc_incs,
                                       int32_t n_bc, const int64_t* pins, int64_t n_pins,
                                       pf_stats* out, double* hist, int32_t hist_cap) {
  if (!h) return PF_ERR_INVALID;
  PF_CUDA(cudaSetDevice(h->device));
  if (scheme < PF_ST || scheme > PF_S3) return fail(h, PF_ERR_INVALID, "unknown scheme");
  h->acc = pf_stats{};
  pf_stats& st = h->acc;
  const pf_config& cfg = h->cfg;
  BcView bc{bc_dofs, bc_offsets, bc_incs, n_bc};
  PF_TRY(set_pmask(h, pins, n_pins));
  std::vector<double> history;
  double r0_u = NAN, r0_d = NAN, last_u_ratio = 0.0;
  PF_CUDA(cudaEventRecord(h->evs0, h->stream));
  double t0 = now_s();
  int nnr = 0;
  PF_TRY(momentum(h, bc, true, &r0_u, &nnr, &last_u_ratio, 0));
  st.n_nr_u += nnr;
  st.wall_u += now_s() - t0;
  double snorm;
  PF_TRY(evo_norm(h, &snorm));
  r0_d = snorm;
  history.push_back(1.0);
  bool converged = snorm <= cfg.res_floor;
  while (!converged) {
    if (st.n_stag >= cfg.max_stag) {
      char buf[128];
      snprintf(buf, sizeof buf, "staggered loop did not converge in %d iterations", cfg.max_stag);
      h->err = buf;
      st.n_hist = (int)std::min<size_t>(history.size(), (size_t)std::max(hist_cap, 0));
      if (hist) std::copy(history.begin(), history.begin() + st.n_hist, hist);
      if (out) *out = st;
      return PF_ERR_CONV_STAGGERED;
    }
    st.n_stag += 1;
    t0 = now_s();
    int nd = 0;
    PF_TRY(evolution(h, scheme, &r0_d, &nd, &st.spd_fallbacks, st.n_stag));
    st.n_nr_d += nd;
    st.wall_d += now_s() - t0;
    t0 = now_s();
    PF_TRY(momentum(h, bc, false, &r0_u, &nnr, &last_u_ratio, st.n_stag));
    st.n_nr_u += nnr;
    st.wall_u += now_s() - t0;
    PF_TRY(evo_norm(h, &snorm));
    const double ratio = snorm / std::max(r0_d, cfg.res_floor);
    history.push_back(ratio);
    converged = snorm <= std::max(cfg.tol_st * r0_d, cfg.res_floor);
  }
  st.final_rd_ratio = st.n_stag ? history.back() : 0.0;
  st.final_ru_ratio = last_u_ratio;
  PF_TRY(commit(h));
  PF_CUDA(cudaEventRecord(h->evs1, h->stream));
  PF_CUDA(cudaStreamSynchronize(h->stream));
  {
    float ms = 0.f;
    PF_CUDA(cudaEventElapsedTime(&ms, h->evs0, h->evs1));
    st.step_ms = ms;
  }
  st.n_hist = (int)std::min<size_t>(history.size(), (size_t)std::max(hist_cap, 0));
  if (hist) std::copy(history.begin(), history.begin() + st.n_hist, hist);
  if (out) *out = st;
  return PF_OK;
}

extern "C" pf_status pf_solve_momentum(pf_handle* h, const int64_t* bc_dofs,
                                       const int64_t* bc_offsets, const double* bc_incs,
                                       int32_t n_bc, double* r0_u, int32_t* n_nr,
                                       double* last_ratio) {
  if (!h) return PF_ERR_INVALID;
  PF_CUDA(cudaSetDevice(h->device));
  h->acc = pf_stats{};
  BcView bc{bc_dofs, bc_offsets, bc_incs, n_bc};
  int nnr = 0;
  double lr = 0.0;
  PF_TRY(momentum(h, bc, true, r0_u, &nnr, &lr, 0));
  PF_CUDA(cudaStreamSynchronize(h->stream));
  if (n_nr) *n_nr = nnr;
  if (last_ratio) *last_ratio = lr;
  return PF_OK;
}

extern "C" pf_status pf_solve_evolution(pf_handle* h, int scheme, const int64_t* pins,
                                        int64_t n_pins, double* r0_d, int32_t* n_nr,
                                        int32_t* spd_fallbacks) {
  if (!h) return PF_ERR_INVALID;
  PF_CUDA(cudaSetDevice(h->device));
  h->acc = pf_stats{};
  PF_TRY(set_pmask(h, pins, n_pins));
  int nd = 0, fb = 0;
  PF_TRY(evolution(h, scheme, r0_d, &nd, &fb));
  PF_CUDA(cudaStreamSynchronize(h->stream));
  if (n_nr) *n_nr = nd;
  if (spd_fallbacks) *spd_fallbacks += fb;
  return PF_OK;
}

extern "C" pf_status pf_evolution_residual_norm(pf_handle* h, const int64_t* pins,
                                                int64_t n_pins, double* out) {
  if (!h) return PF_ERR_INVALID;
  PF_CUDA(cudaSetDevice(h->device));
  PF_TRY(set_pmask(h, pins, n_pins));
  return evo_norm(h, out);
}

extern "C" pf_status pf_commit_step(pf_handle* h) {
  if (!h) return PF_ERR_INVALID;
  PF_CUDA(cudaSetDevice(h->device));
  PF_TRY(commit(h));
  PF_CUDA(cudaStreamSynchronize(h->stream));
  return PF_OK;
}

// ------------------------------------------------------------------------------------------
// operators at the current state
extern "C" pf_status pf_internal_force(pf_handle* h, double* f_out) {
  if (!h) return PF_ERR_INVALID;
  PF_CUDA(cudaSetDevice(h->device));
  PF_TRY(launch_mom_prepare(h, 0));
  PF_TRY(d2h(h, f_out, h->Ru, 2 * (size_t)h->n_nodes));
  PF_CUDA(cudaStreamSynchronize(h->stream));
  return PF_OK;
}

extern "C" pf_status pf_reaction_force(pf_handle* h, const int64_t* nodes, int64_t n,
                                       int component, double* out) {
  if (!h) return PF_ERR_INVALID;
  PF_CUDA(cudaSetDevice(h->device));
  if (component < 0 || component > 1) return fail(h, PF_ERR_INVALID, "component must be 0 or 1");
  for (int64_t i = 0; i < n; ++i)
    if (nodes[i] < 0 || nodes[i] >= h->n_nodes)
      return fail(h, PF_ERR_INDEX, "reaction node outside the mesh");
  PF_TRY(launch_mom_prepare(h, 0));
  PF_TRY(ensure_idx(h, (size_t)n));
  if (n > 0)
    PF_CUDA(cudaMemcpyAsync(h->d_idx, nodes, n * sizeof(long long), cudaMemcpyHostToDevice,
                            h->stream));
  pfb::k_reaction<<<1, 256, 0, h->stream>>>(h->Ru, h->d_idx, n, component,
                                            h->comm ? h->d_red : h->d_scal);
  PF_TRY(launched(h));
  if (h->comm) {  // callers pass their OWNED nodes of the set
    PF_TRY(comm_check(h, h->comm->allreduce(h->d_red, 1, h->stream)));
    PF_CUDA(cudaMemcpyAsync(h->h_scal, h->d_red, sizeof(double), cudaMemcpyDeviceToHost,
                            h->stream));
  }
  PF_CUDA(cudaStreamSynchronize(h->stream));
  *out = h->h_scal[0];
  return PF_OK;
}

extern "C" pf_status pf_momentum_tangent_apply(pf_handle* h, const double* x, double* y,
                                               double* diag) {
  if (!h) return PF_ERR_INVALID;
  PF_CUDA(cudaSetDevice(h->device));
  PF_TRY(launch_mom_prepare(h, 1));  // branch flags and raw diagonal at the current u
  PF_TRY(h2d(h, h->p0u, x, 2 * (size_t)h->n_nodes));
  pfb::CgArgs a = cg_args(h, true);
  a.g = h->geom_apply;
  pfb::k_apply<true><<<(a.g.n_units + 7) / 8, pfb::NT, 0, h->stream>>>(a, h->p0u);
  PF_TRY(launched(h));
  PF_TRY(d2h(h, y, h->qu, 2 * (size_t)h->n_nodes));
  PF_TRY(d2h(h, diag, h->diagu, 2 * (size_t)h->n_nodes));
  PF_CUDA(cudaStreamSynchronize(h->stream));
  return PF_OK;
}

extern "C" pf_status pf_evolution_residual(pf_handle* h, double* r_out) {
  if (!h) return PF_ERR_INVALID;
  PF_CUDA(cudaSetDevice(h->device));
  PF_TRY(launch_evo_prepare(h, 0, 0));
  PF_TRY(d2h(h, r_out, h->Rd, (size_t)h->n_nodes));
  PF_CUDA(cudaStreamSynchronize(h->stream));
  return PF_OK;
}

extern "C" pf_status pf_evolution_tangent_apply(pf_handle* h, int scheme, const double* x,
                                                double* y, double* diag) {
  if (!h) return PF_ERR_INVALID;
  PF_CUDA(cudaSetDevice(h->device));
  if (scheme < PF_ST || scheme > PF_S3) return fail(h, PF_ERR_INVALID, "unknown scheme");
  PF_TRY(launch_evo_prepare(h, 1, scheme));
  PF_TRY(h2d(h, h->p0d, x, (size_t)h->n_nodes));
  pfb::CgArgs a = cg_args(h, false);
  a.g = h->geom_apply;
  pfb::k_apply<false><<<(a.g.n_units + 7) / 8, pfb::NT, 0, h->stream>>>(a, h->p0d);
  PF_TRY(launched(h));
  PF_TRY(d2h(h, y, h->qd, (size_t)h->n_nodes));
  PF_TRY(d2h(h, diag, h->diagd, (size_t)h->n_nodes));
  PF_CUDA(cudaStreamSynchronize(h->stream));
  return PF_OK;
}

extern "C" pf_status pf_refresh_gp(pf_handle* h) {
  if (!h) return PF_ERR_INVALID;
  PF_CUDA(cudaSetDevice(h->device));
  pfb::GpArgs g = gp_args(h);
  pfb::k_refresh_gp<<<cell_grid(h), 128, 0, h->stream>>>(g);
  PF_TRY(launched(h));
  PF_CUDA(cudaStreamSynchronize(h->stream));
  return PF_OK;
}

extern "C" pf_status pf_softening_gate(pf_handle* h, uint8_t* gate_out) {
  if (!h) return PF_ERR_INVALID;
  PF_CUDA(cudaSetDevice(h->device));
  pfb::GpArgs g = gp_args(h);
  g.gate = reinterpret_cast<uint8_t*>(h->scratch);
  pfb::k_gate_extra<<<cell_grid(h), 128, 0, h->stream>>>(g);
  PF_TRY(launched(h));
  PF_CUDA(cudaMemcpyAsync(gate_out, h->scratch, 4 * (size_t)h->n_elems, cudaMemcpyDeviceToHost,
                          h->stream));
  PF_CUDA(cudaStreamSynchronize(h->stream));
  return PF_OK;
}

extern "C" pf_status pf_extra_stiffness(pf_handle* h, int scheme, double* extra_out) {
  if (!h) return PF_ERR_INVALID;
  PF_CUDA(cudaSetDevice(h->device));
  if (scheme < PF_ST || scheme > PF_S3) return fail(h, PF_ERR_INVALID, "unknown scheme");
  pfb::GpArgs g = gp_args(h);
  g.extra = h->scratch;
  g.scheme = scheme;
  pfb::k_gate_extra<<<cell_grid(h), 128, 0, h->stream>>>(g);
  PF_TRY(launched(h));
  PF_TRY(d2h(h, extra_out, h->scratch, 4 * (size_t)h->n_elems));
  PF_CUDA(cudaStreamSynchronize(h->stream));
  return PF_OK;
}

extern "C" pf_status pf_update_active_energy(pf_handle* h, int scheme, const double* dd) {
  if (!h) return PF_ERR_INVALID;
  PF_CUDA(cudaSetDevice(h->device));
  if (scheme < PF_ST || scheme > PF_S3) return fail(h, PF_ERR_INVALID, "unknown scheme");
  if (scheme == PF_ST) return PF_OK;  // schemes.py:162-163
  PF_TRY(h2d(h, h->xd, dd, (size_t)h->n_nodes));
  pfb::GpArgs g = gp_args(h);
  g.dd = h->xd;
  g.scheme = scheme;
  pfb::k_update_energy<<<cell_grid(h), 128, 0, h->stream>>>(g);
  PF_TRY(launched(h));
  PF_CUDA(cudaStreamSynchronize(h->stream));
  return PF_OK;
}

// ------------------------------------------------------------------------------------------
extern "C" pf_status pf_bench_cg(pf_handle* h, int physics, int64_t n_iter, double* ms_out,
                                 int64_t* iters_out) {
  if (!h) return PF_ERR_INVALID;
  PF_CUDA(cudaSetDevice(h->device));
  if (n_iter < 1 || physics < 0 || physics > 3) return fail(h, PF_ERR_INVALID, "bad arguments");
  if (physics == 3) {  // scalar phase-field multigrid PCG (pf_mgs.cuh), fresh hierarchy
    if (!h->mgs.on) return fail(h, PF_ERR_INVALID, "no scalar phase-field hierarchy on this handle");
    PF_TRY(launch_evo_prepare(h, 1, 0));
    int status = 0;
    long long iters = 0;
    PF_TRY(run_mgs(h, h->mgs, &status, &iters, n_iter, 0.0, false));
    float ms = 0.f;
    PF_CUDA(cudaEventElapsedTime(&ms, h->ev0, h->ev1));
    if (ms_out) *ms_out = ms;
    if (iters_out) *iters_out = iters;
    return PF_OK;
  }
  if (physics == 2) {  // multigrid-preconditioned momentum PCG
    if (!h->mgu.on) return fail(h, PF_ERR_INVALID, "no multigrid hierarchy on this handle");
    PF_TRY(launch_mom_prepare(h, 1));
    int status = 0;
    long long iters = 0;
    PF_TRY(run_mg(h, h->mgu, nullptr, &status, &iters, 0, n_iter, 0.0, false, true));
    float ms = 0.f;
    PF_CUDA(cudaEventElapsedTime(&ms, h->ev0, h->ev1));
    if (ms_out) *ms_out = ms;
    if (iters_out) *iters_out = iters;
    return PF_OK;
  }
  const bool mom = physics == 0;
  if (mom) PF_TRY(launch_mom_prepare(h, 1));
  else PF_TRY(launch_evo_prepare(h, 1, 0));
  pfb::CgArgs a = cg_args(h, mom);
  a.rtol = 0.0;  // never converges: exactly n_iter iterations
  a.maxiter = n_iter;
  void* args[] = {&a};
  const void* fn = cg_kernel(h, mom);
  PF_CUDA(cudaEventRecord(h->ev0, h->stream));
  PF_CUDA(cudaLaunchCooperativeKernel(fn, dim3(mom ? h->cg_grid : h->cg_grid_evo),
                                      dim3(pfb::CG_NT), args,
                                      cg_smem(h, mom), h->stream));
  PF_TRY(launched(h));
  PF_CUDA(cudaEventRecord(h->ev1, h->stream));
  PF_CUDA(cudaStreamSynchronize(h->stream));
  float ms = 0.f;
  PF_CUDA(cudaEventElapsedTime(&ms, h->ev0, h->ev1));
  if (ms_out) *ms_out = ms;
  if (iters_out) *iters_out = h->h_cgres->iters;
  if (h->h_cgres->status == pfb::CG_NAN) return fail(h, PF_ERR_SINGULAR, "non-finite residual");
  return PF_OK;
}

// Average device time of one fine-level multigrid march on the current hierarchy and state,
// re-launched `reps` times outside the solve graph (CUDA events on the handle's stream; a kernel
// inside the conditional solve graph cannot be event-timed or seen by ncu).  which: 0 / 1 / 2
// the momentum hierarchy's fine residual, smoothing and PCG-direction marches; 10 / 11 / 12 the
// same of the scalar phase-field hierarchy.  bytes_out: the kernel's algorithmic bytes per launch
// (compulsory traffic of its inputs and outputs).
extern "C" pf_status pf_bench_mg_kernel(pf_handle* h, int which, int reps, double* ms_out,
                                        double* bytes_out) {
  if (!h) return PF_ERR_INVALID;
  PF_CUDA(cudaSetDevice(h->device));
  if (reps < 1) return fail(h, PF_ERR_INVALID, "pf_bench_mg_kernel: reps < 1");
  const double n = h->n_nodes, e = h->n_elems;
  double bytes = 0.0;
  auto run = [&](auto&& launch) -> pf_status {
    launch();  // warm
    PF_CUDA(cudaEventRecord(h->ev0, h->stream));
    for (int k = 0; k < reps; ++k) launch();
    PF_CUDA(cudaEventRecord(h->ev1, h->stream));
    PF_CUDA(cudaStreamSynchronize(h->stream));
    PF_CUDA(cudaGetLastError());
    return PF_OK;
  };
  cudaStream_t s = h->stream;
  if (which >= 0 && which <= 2) {
    if (!h->mgu.on || !h->mgu.built) return fail(h, PF_ERR_INVALID, "no built momentum hierarchy");
    MgInst& M = h->mgu;
    pfb::MgArgs A = M.A;
    A.use_cond = 0;
    const double n1 = A.L[1].m.n_nodes;
    if (which == 0) {
      bytes = 56.0 * n + e;  // r, D^-1 (16 B), d (8 B), t (16 B); branch bits 1 B per cell
      PF_TRY(run([&] { pfb::k_mg_fine_resid<<<M.gf, pfb::MG_NT, 0, s>>>(A); }));
    } else if (which == 1) {
      bytes = 56.0 * n + 16.0 * n1 + e;  // r, D^-1, d, z; level-1 correction; bits
      PF_TRY(run([&] { pfb::k_mg_fine_smooth<<<M.gf, pfb::MG_NT, 0, s>>>(A); }));
    } else {
      bytes = 88.0 * n + e;  // z, p_old, d, D^-1, p_new, q; bits
      PF_TRY(run([&] { pfb::k_mg_pcg<<<M.gf, pfb::MG_NT, 0, s>>>(A, M.gf); }));
    }
  } else if (which >= 10 && which <= 12) {
    if (!h->mgs.on || h->mgs.setups == 0) return fail(h, PF_ERR_INVALID, "no built phase-field hierarchy");
    MgsInst& M = h->mgs;
    pfb::MgsArgs A = M.A;
    A.use_cond = 0;
    const double n1 = A.L[1].m.n_nodes;
    if (which == 10) {
      bytes = 24.0 * n + 32.0 * e;  // r, D^-1, t (8 B); b per Gauss point (32 B per cell)
      PF_TRY(run([&] { pfb::k_mgs_fine_resid<<<M.gfr, pfb::MG_NT, 0, s>>>(A); }));
    } else if (which == 11) {
      bytes = 24.0 * n + 8.0 * n1 + 32.0 * e;  // r, D^-1, z; level-1 correction; b
      PF_TRY(run([&] { pfb::k_mgs_fine_smooth<<<M.gf, pfb::MG_NT, 0, s>>>(A); }));
    } else {
      bytes = 40.0 * n + 32.0 * e;  // z, p_old, D^-1, p_new, q; b
      PF_TRY(run([&] { pfb::k_mgs_pcg<<<M.gf, pfb::MG_NT, 0, s>>>(A, M.gf); }));
    }
  } else {
    return fail(h, PF_ERR_INVALID, "pf_bench_mg_kernel: unknown kernel");
  }
  float ms = 0.f;
  PF_CUDA(cudaEventElapsedTime(&ms, h->ev0, h->ev1));
  if (ms_out) *ms_out = ms / reps;
  if (bytes_out) *bytes_out = bytes;
  return PF_OK;
}

extern "C" pf_status pf_mg_info(pf_handle* h, int32_t* n_levels, int32_t* n_grid,
                                int32_t* dense, int64_t* setups, double* omega) {
  if (!h) return PF_ERR_INVALID;
  PF_CUDA(cudaSetDevice(h->device));
  if (setups) *setups = h->mgu.setups;
  if (n_levels) *n_levels = h->mgu.on ? h->mgu.A.n_levels : 0;
  if (n_grid) *n_grid = h->mgu.on ? h->mgu.A.n_tail : 0;
  if (dense) *dense = h->mgu.on ? h->mgu.A.dense : 0;
  if (!h->mgu.on || !omega) return PF_OK;
  PF_TRY(launch_mom_prepare(h, 1));
  int status = 0;
  long long iters = 0;
  PF_TRY(run_mg(h, h->mgu, nullptr, &status, &iters, 1));
  PF_CUDA(cudaMemcpy(omega, h->mgu.A.ctl->omega, h->mgu.A.n_levels * sizeof(double),
                     cudaMemcpyDeviceToHost));
  return PF_OK;
}

extern "C" pf_status pf_solver_kinds(pf_handle* h, int32_t* momentum, int32_t* phase_field) {
  if (!h) return PF_ERR_INVALID;
  if (momentum) *momentum = h->mgu.on ? 2 : (h->sr_mom ? 1 : 0);
  if (phase_field)
    *phase_field = h->mgs.on && !h->comm   ? 4
                   : h->mgd.on && !h->comm ? 3
                   : (h->sr_evo && !h->comm && !h->split ? (h->st_evo ? 2 : 1) : 0);
  return PF_OK;
}

extern "C" pf_status pf_device_info(pf_handle* h, int32_t* cg_grid, int32_t* sm_count,
                                    int64_t* l2_bytes) {
  if (!h) return PF_ERR_INVALID;
  if (cg_grid) *cg_grid = h->cg_grid;
  if (sm_count) *sm_count = h->sm_count;
  if (l2_bytes) *l2_bytes = h->l2_bytes;
  return PF_OK;
}

extern "C" pf_status pf_flush_l2(pf_handle* h) {
  if (!h) return PF_ERR_INVALID;
  PF_CUDA(cudaSetDevice(h->device));
  if (!h->flushbuf) {
    h->flush_n = (size_t)std::max<long long>(2 * h->l2_bytes, 256LL << 20) / sizeof(double);
    PF_CUDA(cudaMalloc((void**)&h->flushbuf, h->flush_n * sizeof(double)));
  }
  pfb::k_flush<<<h->sm_count * 4, 256, 0, h->stream>>>(h->flushbuf, (long long)h->flush_n, 1.0);
  PF_TRY(launched(h));
  PF_CUDA(cudaStreamSynchronize(h->stream));
  return PF_OK;
}

extern "C" pf_status pf_synchronize(pf_handle* h) {
  if (!h) return PF_ERR_INVALID;
  PF_CUDA(cudaSetDevice(h->device));
  PF_CUDA(cudaStreamSynchronize(h->stream));
  return PF_OK;
}
