// pf_march.cuh — barrier-free register-marching phase A of the persistent PCG.
//
// A work unit is (strip, row block): a warp owns TXW = 30 node columns (lanes 1..30; lanes 0
// and 31 carry the halo columns) and marches up node rows r0-1 .. r1 keeping two node rows in
// registers.  Lane l evaluates cell (col_l, cj) from its own and lane l+1's nodes (shuffle),
// and each node's four cell contributions arrive in the reference's element order
//     ((c2 of (i-1,j-1) + c3 of (i,j-1)) + c1 of (i-1,j)) + c0 of (i,j)
// (np.add.at / COO->CSR order, assembly.py:188, :195-197), so results are bit-identical to the
// tile formulation.  No shared memory, no CTA barriers; the next row's loads are issued before
// the current row's FP64 work, so every warp keeps a row of loads in flight.  The x update of
// the CG moved to the streaming phase B; phase A only reads p_{k-1}, r, D^-1 (and d) and writes
// p_k and q.
//
// The slit (meshing.py:126-138): node row R holds lower-face nodes, and for columns in
// [notch_lo, notch_hi) a second, upper-face set (the duplicates) used as bottom corners by
// cell row R.  Rows with variable extents (L-panel, meshing.py:179-192) come from the row
// tables (broadcast __ldg loads, L1-resident).
#pragma once

namespace pfb {

constexpr int TXW = 30;  // owned columns per warp strip

__device__ __forceinline__ double shfl_dn(double v) { return __shfl_down_sync(0xffffffffu, v, 1); }
__device__ __forceinline__ double shfl_up(double v) { return __shfl_up_sync(0xffffffffu, v, 1); }
__device__ __forceinline__ double2 shfl_dn(double2 v) {
  return make_double2(shfl_dn(v.x), shfl_dn(v.y));
}
__device__ __forceinline__ double2 shfl_up(double2 v) {
  return make_double2(shfl_up(v.x), shfl_up(v.y));
}

// Element tangent-vector product K_e(u, d) p_e on a uniform cell, grouped by the tensor-product
// structure: each derivative takes two distinct values per cell, and the back-projection sums
// Gauss-point pairs first (~130 FP64 operations per cell, no division).
__device__ __forceinline__ void mom_cell_fast(const Consts& C, const double2 (&pc)[4],
                                              const double (&dc)[4], unsigned flags,
                                              double2 (&f)[4]) {
  const double bx = pc[1].x - pc[0].x, tx = pc[2].x - pc[3].x;
  const double by = pc[1].y - pc[0].y, ty = pc[2].y - pc[3].y;
  const double lx = pc[3].x - pc[0].x, rx = pc[2].x - pc[1].x;
  const double ly = pc[3].y - pc[0].y, ry = pc[2].y - pc[1].y;
  const double uxx_lo = C.Px * bx + C.Mx * tx, uxx_hi = C.Mx * bx + C.Px * tx;
  const double uyx_lo = C.Px * by + C.Mx * ty, uyx_hi = C.Mx * by + C.Px * ty;
  const double uxy_l = C.Py * lx + C.My * rx, uxy_r = C.My * lx + C.Py * rx;
  const double uyy_l = C.Py * ly + C.My * ry, uyy_r = C.My * ly + C.Py * ry;
  const double exx[4] = {uxx_lo, uxx_lo, uxx_hi, uxx_hi};
  const double eyy[4] = {uyy_l, uyy_r, uyy_r, uyy_l};
  const double gxy[4] = {uxy_l + uyx_lo, uxy_r + uyx_lo, uxy_r + uyx_hi, uxy_l + uyx_hi};
  double sxx[4], syy[4], sxy[4];
#pragma unroll
  for (int g = 0; g < 4; ++g) {
    const double dg = C.N[g][0] * dc[0] + C.N[g][1] * dc[1] + C.N[g][2] * dc[2] +
                      C.N[g][3] * dc[3];
    const double om = 1.0 - dg;
    const double gg = om * om + C.eta;
    const double tr = exx[g] + eyy[g];
    const double a = gg * C.two_mu;
    const double kv = ((flags >> g) & 1u) ? gg * C.k : C.k;
    const double t3 = tr * C.third;
    sxx[g] = a * (exx[g] - t3) + kv * tr;
    syy[g] = a * (eyy[g] - t3) + kv * tr;
    sxy[g] = (gg * C.mu) * gxy[g];
  }
  const double xx01 = sxx[0] + sxx[1], xx23 = sxx[2] + sxx[3];
  const double yy03 = syy[0] + syy[3], yy12 = syy[1] + syy[2];
  const double xy01 = sxy[0] + sxy[1], xy23 = sxy[2] + sxy[3];
  const double xy03 = sxy[0] + sxy[3], xy12 = sxy[1] + sxy[2];
  const double axx = C.Pxw * xx01 + C.Mxw * xx23, bxx = C.Mxw * xx01 + C.Pxw * xx23;
  const double cyy = C.Pyw * yy03 + C.Myw * yy12, dyy = C.Myw * yy03 + C.Pyw * yy12;
  const double axy = C.Pxw * xy01 + C.Mxw * xy23, bxy = C.Mxw * xy01 + C.Pxw * xy23;
  const double cxy = C.Pyw * xy03 + C.Myw * xy12, dxy = C.Myw * xy03 + C.Pyw * xy12;
  f[0] = make_double2(-axx - cxy, -cyy - axy);
  f[1] = make_double2(axx - dxy, -dyy + axy);
  f[2] = make_double2(bxx + dxy, dyy + bxy);
  f[3] = make_double2(-bxx + cxy, cyy - bxy);
}

// ---- cp.async staging (single-reduction march): a lane's next node row is copied L2 -> smem
// without register staging (zero-fill for absent values), so the six vectors the SR node update
// needs do not occupy registers while in flight
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool valid) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(gmem),
               "r"(valid ? 16 : 0));
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, bool valid) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(sa), "l"(gmem),
               "r"(valid ? 8 : 0));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::); }
__device__ __forceinline__ void cp_async_wait_1() { asm volatile("cp.async.wait_group 1;\n" ::); }
template <bool MOM>
__device__ __forceinline__ void cp_async_t(typename Node<MOM>::T* smem, const double* g, int id,
                                           bool valid) {
  const int cid = valid ? id : 0;
  if constexpr (MOM) cp_async16(smem, g + 2 * (size_t)cid, valid);
  else cp_async8(smem, g + cid, valid);
}

template <bool MOM>
struct SrStage {  // one node row of one warp (lane-private columns)
  using T = typename Node<MOM>::T;
  T r[32], di[32], po[32], x[32], s[32], wo[32];
  double d[32];
};
constexpr int SR_SLOTS = 3;  // per warp: two alternating node rows, the slit-duplicate row
extern __shared__ __align__(16) unsigned char pf_dyn_smem[];
template <bool MOM>
__device__ __forceinline__ SrStage<MOM>& sr_slot(int which) {
  return reinterpret_cast<SrStage<MOM>*>(pf_dyn_smem)[(threadIdx.x >> 5) * SR_SLOTS + which];
}

template <bool MOM>
struct RawNode {
  using T = typename Node<MOM>::T;
  T r, di, po, x;
  double d;
  int id;
  int slot;  // SR: staging slot of this row (sr_slot)
  int pend;  // SR: a younger row's copies were committed after this row's (wait_group 1)
};

// XUPD (lazy solution update): the owner of a node also loads x so that finish_node can apply
// x += alpha_{k-1} p_{k-1} with the p_{k-1} the march reads anyway (phase B then no longer
// streams p and x: 32 B per node and iteration less)
template <bool MOM, bool APPLY, bool XUPD = false, int SR = 0>
__device__ __forceinline__ void fetch_node(const CgArgs& a, const double* __restrict__ pold,
                                           bool first, int id, RawNode<MOM>& w,
                                           bool xown = false, const SrScal* sp = nullptr) {
  using N_ = Node<MOM>;
  w.id = id;
  if (id >= 0) {
    if constexpr (SR != 0) {
      using B = SrBuf<SR == 2>;
      SrStage<MOM>& st = sr_slot<MOM>(w.slot);
      const int ln = threadIdx.x & 31;
      const bool upd = !sp->first, old = upd && !sp->fresh;
      cp_async_t<MOM>(&st.r[ln], B::rin(a), id, true);
      cp_async_t<MOM>(&st.di[ln], a.dinv, id, true);
      cp_async_t<MOM>(&st.wo[ln], B::win(a), id, upd);
      cp_async_t<MOM>(&st.s[ln], B::sin(a), id, old);
      cp_async_t<MOM>(&st.po[ln], a.pc, id, old && xown);
      cp_async_t<MOM>(&st.x[ln], a.x, id, upd && xown);
      if constexpr (MOM) cp_async8(&st.d[ln], a.d + id, true);
      cp_async_commit();
    } else if (APPLY) {
      w.po = N_::ld_ro(pold, id);
    } else {
      w.r = N_::ld_cg(a.r, id);
      w.di = N_::ld_ro(a.dinv, id);
      if (!first) w.po = N_::ld_cg(pold, id);
      if (XUPD && !first && xown) w.x = N_::ld_cg(a.x, id);
    }
    if constexpr (MOM && SR == 0) w.d = __ldg(a.d + id);
  }
}

// p_k = D^-1 r + beta p_{k-1}; the owner stores it (and, XUPD, x += alpha_{k-1} p_{k-1}).
// SR (1 even / 2 odd pass): the single-reduction node update (pf_cg.cuh SrBuf); returns u = D^-1 r_new, the vector multiplied.
template <bool MOM, bool APPLY, bool XUPD = false, int SR = 0>
__device__ __forceinline__ typename Node<MOM>::T finish_node(const RawNode<MOM>& w, bool first,
                                                             double beta, bool own,
                                                             double* __restrict__ pnew,
                                                             double* __restrict__ x = nullptr,
                                                             double xalpha = 0.0,
                                                             const SrScal* sp = nullptr,
                                                             double* rr = nullptr,
                                                             double* gam = nullptr,
                                                             const CgArgs* ap = nullptr) {
  using N_ = Node<MOM>;
  if (w.id < 0) return N_::zero();
  if constexpr (SR != 0) {
    using T = typename N_::T;
    using B = SrBuf<SR == 2>;
    const CgArgs& a = *ap;
    const int ln = threadIdx.x & 31;
    if (w.pend) cp_async_wait_1();
    else cp_async_wait_all();
    const SrStage<MOM>& st = sr_slot<MOM>(w.slot);
    const T r0 = st.r[ln], di = st.di[ln];
    const T uo = N_::mul(di, r0);
    if (sp->first) {
      if (own) {
        N_::st(B::rout(a), w.id, r0);
        *rr += N_::dot(r0, r0);
        *gam += N_::dot(r0, uo);
      }
      return uo;
    }
    const T sv = N_::axpy(sp->beta, st.s[ln], st.wo[ln]);  // s = w + beta s
    const T rv = N_::axpy(-sp->alpha, sv, r0);             // r -= alpha s
    const T u = N_::mul(di, rv);
    if (own) {
      const T pv = N_::axpy(sp->beta, st.po[ln], uo);      // p = D^-1 r_old + beta p
      N_::st(a.pc, w.id, pv);
      N_::st(a.x, w.id, N_::axpy(sp->alpha, pv, st.x[ln]));  // x += alpha p
      N_::st(B::sout(a), w.id, sv);
      N_::st(B::rout(a), w.id, rv);
      *rr += N_::dot(rv, rv);
      *gam += N_::dot(rv, u);
    }
    return u;
  }
  if (APPLY) return w.po;
  typename N_::T p = N_::mul(w.di, w.r);
  if (!first) p = N_::axpy(beta, w.po, p);
  if (own) N_::st(pnew, w.id, p);
  if (XUPD && !first && own) N_::st(x, w.id, N_::axpy(xalpha, w.po, w.x));
  return p;
}

// the slit row's upper-face (duplicate) nodes of one warp, parked in shared memory so the march
// does not carry them in registers through every row
template <bool MOM>
struct DupRow {
  typename Node<MOM>::T p[32];
  double d[32];
  int id[32];
  unsigned fb[32];
  // 32-row windows of the node-row / cell-row tables (refilled by one coalesced load every 32
  // rows): the per-row lookups are shared-memory broadcasts instead of dependent global loads
  int4 nwin[32], ewin[32];
};

template <bool MOM, bool APPLY, bool XUPD = false, int SR = 0>
__device__ __forceinline__ void march_unit(const CgArgs& a, const MarchGeom& G, int unit,
                                           bool first, double beta,
                                           const double* __restrict__ pold,
                                           double* __restrict__ pnew, double& pq,
                                           DupRow<MOM>& dup, double xalpha = 0.0,
                                           const SrScal* sp = nullptr, double* rr = nullptr,
                                           double* gam = nullptr) {
  using N_ = Node<MOM>;
  using T = typename N_::T;
  const DMesh& m = a.m;
  const Consts& C = a.C;
  const int lane = threadIdx.x & 31;
  const int strip = unit % G.n_strips;
  const int r0 = (unit / G.n_strips) * G.rows_per_unit;
  const int r1 = min(r0 + G.rows_per_unit, m.ny + 1);
  const int col = strip * TXW - 1 + lane;
  const bool lane_own = lane >= 1 && lane <= TXW;
  const int R = m.notch_row;
  const bool dupcol = R >= 0 && col >= m.notch_lo && col < m.notch_hi;
  int nbase = -1000000, ebase = -1000000;  // warp-uniform window bases
  auto nid = [&](int j) -> int {
    if (j < 0 || j > m.ny) return -1;
    if (j - nbase >= 32 || j < nbase) {  // warp-uniform refill
      __syncwarp();
      nbase = j;
      const int jj = j + lane;
      dup.nwin[lane] = jj <= m.ny ? __ldg(m.nrow + jj) : make_int4(0, 0, 0, 0);
      __syncwarp();
    }
    const int4 rw = dup.nwin[j - nbase];
    return (col >= rw.x && col < rw.y) ? rw.z + (col - rw.x) : -1;
  };
  // d and D^-1 of a finished row (SR: still in its staging slot)
  auto node_d = [&](const RawNode<MOM>& v) -> double {
    if constexpr (!MOM) return 0.0;
    else if constexpr (SR != 0) return v.id >= 0 ? sr_slot<MOM>(v.slot).d[lane] : 0.0;
    else return v.d;
  };
  auto node_fb = [&](const RawNode<MOM>& v) -> unsigned {
    if (APPLY || v.id < 0) return 0u;
    if constexpr (SR != 0) return N_::freebits(sr_slot<MOM>(v.slot).di[lane]);
    else return N_::freebits(v.di);
  };
  // loads and parks the duplicate row (warp-uniform call)
  auto load_dup = [&](bool own) {
    RawNode<MOM> wd;
    wd.slot = 2;
    wd.pend = 0;
    fetch_node<MOM, APPLY, XUPD, SR>(a, pold, first,
                                     dupcol ? m.dup_start + (col - m.notch_lo) : -1, wd, own, sp);
    dup.p[lane] = finish_node<MOM, APPLY, XUPD, SR>(wd, first, beta, own, pnew, a.x, xalpha, sp,
                                                    rr, gam, &a);
    dup.d[lane] = node_d(wd);
    dup.id[lane] = wd.id;
    dup.fb[lane] = node_fb(wd);
    __syncwarp();
  };

  // lower row (cj) state
  T p_lo;
  double d_lo;
  int id_lo;
  unsigned fb_lo;
  bool lo_slit;
  // SR stages node rows in shared memory two rows ahead: w = the row finished next, wn = the
  // row after it (already in flight); a row's slot is refilled right after it is finished.
  // The register path (SR == 0) keeps one row of loads in flight in w.
  RawNode<MOM> w, wn;
  w.slot = 0;
  w.pend = 0;
  wn.slot = 1;
  wn.pend = 0;
  fetch_node<MOM, APPLY, false, SR>(a, pold, first, nid(r0 - 1), w, false, sp);
  if constexpr (SR != 0) {
    fetch_node<MOM, APPLY, XUPD, SR>(a, pold, first, nid(r0), wn, lane_own && r0 < r1, sp);
    w.pend = 1;
  }
  p_lo = finish_node<MOM, APPLY, false, SR>(w, first, beta, false, pnew, nullptr, 0.0, sp, rr,
                                            gam, &a);
  d_lo = node_d(w);
  id_lo = w.id;
  fb_lo = node_fb(w);
  lo_slit = (r0 - 1 == R);
  if (lo_slit) load_dup(false);
  if constexpr (SR != 0) {
    const int fs = w.slot;
    w = wn;
    wn.slot = fs;
    w.pend = 0;
    if (r0 + 1 <= r1) {
      fetch_node<MOM, APPLY, XUPD, SR>(a, pold, first, nid(r0 + 1), wn, lane_own && r0 + 1 < r1,
                                       sp);
      w.pend = 1;
    }
  } else {
    fetch_node<MOM, APPLY, XUPD, SR>(a, pold, first, nid(r0), w, lane_own && r0 < r1, sp);
  }
  // cell-row data (branch bits / Newton coefficients) are prefetched one row ahead too
  auto cell_id = [&](int cj) -> int {
    if (cj < 0 || cj >= m.ny) return -1;
    if (cj - ebase >= 32 || cj < ebase) {  // warp-uniform refill
      __syncwarp();
      ebase = cj;
      const int jj = cj + lane;
      dup.ewin[lane] = jj < m.ny ? __ldg(m.erow + jj) : make_int4(0, 0, 0, 0);
      __syncwarp();
    }
    if (lane >= 31) return -1;
    const int4 er = dup.ewin[cj - ebase];
    return (col >= er.x && col < er.y) ? er.z + (col - er.x) : -1;
  };
  int eid_n = cell_id(r0 - 1);
  unsigned fl_n = 0u;
  double bq_n[4] = {0.0, 0.0, 0.0, 0.0};
  auto fetch_cell = [&](int eid) {
    if (eid < 0) return;
    if constexpr (MOM) fl_n = __ldg(a.flags + eid);
    else load4(a.b, eid, bq_n);
  };
  fetch_cell(eid_n);
  T acc_lo = N_::zero();
  for (int cj = r0 - 1; cj < r1; ++cj) {
    const int jh = cj + 1;
    const bool hi_own = lane_own && jh >= r0 && jh < r1;
    const T p_hi = finish_node<MOM, APPLY, XUPD, SR>(w, first, beta, hi_own, pnew, a.x, xalpha, sp,
                                                     rr, gam, &a);
    const double d_hi = node_d(w);
    const int id_hi = w.id;
    const unsigned fb_hi = node_fb(w);
    const bool hi_slit = (jh == R);
    if constexpr (SR != 0) {  // the finished row's slot takes row jh + 2
      const int fs = w.slot;
      w = wn;
      wn.slot = fs;
      w.pend = 0;
      if (jh + 2 <= r1) {
        fetch_node<MOM, APPLY, XUPD, SR>(a, pold, first, nid(jh + 2), wn,
                                         lane_own && jh + 2 < r1, sp);
        w.pend = 1;
      }
    } else if (jh + 1 <= r1) {  // prefetch
      fetch_node<MOM, APPLY, XUPD, SR>(a, pold, first, nid(jh + 1), w, lane_own && jh + 1 < r1,
                                       sp);
    }
    const int eid = eid_n;
    const unsigned fl = fl_n;
    double bq[4] = {bq_n[0], bq_n[1], bq_n[2], bq_n[3]};
    eid_n = cell_id(cj + 1);
    fetch_cell(eid_n);
    // ---- cell (col, cj)
    const bool use_dup = lo_slit && dupcol;
    const T b0 = use_dup ? dup.p[lane] : p_lo;
    const T b1 = shfl_dn(b0);
    const T t2 = shfl_dn(p_hi);
    T f[4];
    if constexpr (MOM) {
      const double e0 = use_dup ? dup.d[lane] : d_lo;
      const double e1 = shfl_dn(e0);
      const double e2 = shfl_dn(d_hi);
      f[0] = f[1] = f[2] = f[3] = make_double2(0.0, 0.0);
      if (eid >= 0) {
        const double2 pc[4] = {b0, b1, t2, p_hi};
        const double dc[4] = {e0, e1, e2, d_hi};
        mom_cell_fast(C, pc, dc, fl, f);
      }
    } else {
      f[0] = f[1] = f[2] = f[3] = 0.0;
      if (eid >= 0) {
        const double pc[4] = {b0, b1, t2, p_hi};
        evo_cell_apply(C, pc, bq, f);
      }
    }
    // ---- node row cj complete: ((c2 + c3) + c1 from the left) + c0 own
    const T c1l = shfl_up(f[1]);
    const T c2l = shfl_up(f[2]);
    if (lane_own && cj >= r0) {
      if (use_dup) {
        if (id_lo >= 0) {  // lower face: cells below only
          T qv = acc_lo;
          if (!APPLY) {
            qv = N_::maskb(qv, fb_lo);
            if (node_owned(m, id_lo)) pq += N_::dot(p_lo, qv);
          }
          N_::st(SR == 0 ? a.q : SrBuf<SR == 2>::wout(a), id_lo, qv);
        }
        const int idd = dup.id[lane];
        if (idd >= 0) {  // upper face: cells above only
          T qv = add_t(c1l, f[0]);
          if (!APPLY) {
            qv = N_::maskb(qv, dup.fb[lane]);
            if (node_owned(m, idd)) pq += N_::dot(dup.p[lane], qv);
          }
          N_::st(SR == 0 ? a.q : SrBuf<SR == 2>::wout(a), idd, qv);
        }
      } else if (id_lo >= 0) {
        T qv = add_t(add_t(acc_lo, c1l), f[0]);
        if (!APPLY) {
          qv = N_::maskb(qv, fb_lo);
          if (node_owned(m, id_lo)) pq += N_::dot(p_lo, qv);
        }
        N_::st(SR == 0 ? a.q : SrBuf<SR == 2>::wout(a), id_lo, qv);
      }
    }
    acc_lo = add_t(c2l, f[3]);
    if (hi_slit) {  // warp-uniform; the old duplicate row was consumed above
      __syncwarp();
      load_dup(hi_own);
    }
    p_lo = p_hi;
    d_lo = d_hi;
    id_lo = id_hi;
    fb_lo = fb_hi;
    lo_slit = hi_slit;
  }
}

inline MarchGeom make_march_geom(int nx, int ny, int resident_warps, int min_rows = 4) {
  // At most one unit per resident warp: phase A lasts as long as its busiest warp, so the row
  // blocks per strip are floor(warps / strips).  (A ceil split that leaves some warps with two
  // units doubles the phase: 8192^2 had 2466 units for 2368 warps.)  Units never cross a strip:
  // the 8 warps of a CTA march 8 adjacent strips in lockstep and share their halo columns in L2
  // (runs laid end to end over the strips balanced better but measured slower).
  MarchGeom g;
  g.n_strips = (nx + 1 + TXW - 1) / TXW;
  int blocks = resident_warps / g.n_strips;
  blocks = blocks < 1 ? 1 : blocks;
  int rows = (ny + 1 + blocks - 1) / blocks;
  rows = rows < min_rows ? min_rows : rows;
  if (rows > ny + 1) rows = ny + 1;
  g.rows_per_unit = rows;
  g.n_row_blocks = (ny + 1 + rows - 1) / rows;
  g.n_units = g.n_strips * g.n_row_blocks;
  return g;
}

}  // namespace pfb
