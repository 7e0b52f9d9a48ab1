"""Benchmark: load steps of BASELINE configs[4] (8192^2 multi-crack biaxial, 201 M DOFs, FP64).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--case cfg5] [--scheme S1]

Workload: the largest BASELINE configuration that fits one B200 (tier rule: BASELINE's metric
names no config) -- config 5, 1 m square, 8192 x 8192 Q4 cells (67.1 M nodes, 201 M DOFs),
256 seeded pre-cracks, biaxial loading, scheme S1.  A "step" is one load step
(``staggered_step``, reference schemes.py:332-392) of the case's own schedule: W untimed warm-up
load steps advance the state, then K load steps are timed.  ``--case cfg2`` gives round 1's
512 x 512 line (a secondary measurement).

* ``value``   -- DOF-iterations/s (SURVEY.md §8(d) reading 1a: 3*N_nodes * sum n_stag / time),
  device-resident state built on the device (pf_init_state: zero state + pre-cracks), CUDA events
  on the solver stream around each load step.  cfg5's working set (~25 GB) is far beyond L2, so
  no flush is needed between steps; L2-sized cases (cfg2) flush 256 MiB before every step.
* ``e2e``     -- the same metric through the reference-facing drop-in
  ``paper_2209_07969_b200.schemes.staggered_step`` with a HOST SolverState: every step uploads
  the load step's inputs (u, d, d_prev, gp.psi_max) and downloads the whole state including
  gp.strain / gp.tr_eps, all inside the timed region (host wall clock).  ``e2e.pageable`` repeats
  a short sample with a reference-style state of ordinary numpy arrays.
* ``roofline``-- the dominant kernel of the step: its algorithmic bytes per launch
  / its average launch time, timed with CUDA events on the solver stream after the timed region
  (pf_bench_mg_kernel re-launches it on the final state: inside the solve graph a single kernel
  cannot be event-timed), against MEASURED_PEAKS.json; ``traffic`` = its DRAM bytes per launch
  from the committed ``ncu --set full`` capture (profiles/).
* ``cpu_baseline`` -- the CPU oracle port (oracle/phasefield_oracle.py, SuperLU like the
  reference default) on a bounded sample: config 5 cannot be set up on a CPU (the reference's
  Discretization alone needs ~120 GB), so the sample is config 2's first load step.
* ``--gpus N`` (torchrun, one process per GPU) -- the same problem split into N row strips
  (``dist.StripSession``: NCCL halo rows + all-reduces), value = global DOF-iterations /
  max-over-ranks device time.
* ``--impl reference`` -- the reference algorithm on the CPU (the oracle port; the Python
  reference does not travel to the GPU box): config 5 is not runnable on a CPU, so the line
  carries ``value: null`` with the reason, plus a ``secondary`` measurement on config 2 with the
  same W untimed warm-up steps and the following load steps timed (time budget).
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "DOF-iterations/s of staggered solve (FP64)"


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """SM clocks / throttle reasons sampled DURING the timed region: NVML polled every 5 ms from a
    thread; `nvidia-smi -lms 200` when NVML is not importable."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")
    NAMES = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.nvml = None
        self.lines = []
        self.stop = threading.Event()

    def __enter__(self):
        try:
            import pynvml as nv

            nv.nvmlInit()
            vis = os.environ.get("CUDA_VISIBLE_DEVICES")
            idx = int(vis.split(",")[self.index]) if vis and vis.split(",")[0].isdigit() else self.index
            self.handle = nv.nvmlDeviceGetHandleByIndex(idx)
            self.nvml = nv
            self.bits = (nv.nvmlClocksEventReasonHwSlowdown, nv.nvmlClocksEventReasonHwThermalSlowdown,
                         nv.nvmlClocksEventReasonSwThermalSlowdown, nv.nvmlClocksEventReasonSwPowerCap)
            self.t = threading.Thread(target=self._poll, daemon=True)
            self.t.start()
            return self
        except Exception:  # no NVML: nvidia-smi
            self.nvml = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except (OSError, FileNotFoundError):
            self.proc = None
        return self

    def _poll(self):
        nv, h = self.nvml, self.handle
        while not self.stop.is_set():
            try:
                sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
                rs = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                flags = ["Active" if rs & b else "Not Active" for b in self.bits]
                self.lines.append(", ".join([str(sm), str(mx), "0"] + flags))
            except Exception:
                return
            self.stop.wait(0.005)

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        self.stop.set()
        if self.nvml is not None:
            self.t.join(timeout=1.0)
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(self.NAMES, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        src = "nvml (5 ms poll)" if self.nvml is not None else "nvidia-smi -lms 200"
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0,
                    "source": src}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": float(max(mx)),
                "reasons": sorted(reasons), "samples": len(sm), "source": src}


# -------------------------------------------------------------------------------------------
def host_initial_state(dp, case, pinned: bool):
    """The case's initial SolverState on the host: zeros, d = d_prev = 1 at the pre-crack nodes
    (configs.precrack_nodes_grid / precrack_nodes)."""
    from paper_2209_07969_b200 import _native as N
    from paper_2209_07969_b200 import configs as C
    from paper_2209_07969_b200.assembly import GaussPointState
    from paper_2209_07969_b200.schemes import SolverState

    nn, ne = dp.layout.n_nodes, dp.layout.n_elems

    def z(shape):
        a = N.PINNED.empty(shape) if pinned else np.empty(shape)
        a[...] = 0.0
        return a

    gp = GaussPointState(strain=z((ne, 4, 4)), tr_eps=z((ne, 4)), tr_eps_plus=z((ne, 4)),
                         dev_dot_dev=z((ne, 4)), psi_plus=z((ne, 4)), psi_max=z((ne, 4)))
    st = SolverState(u=z(2 * nn), d=z(nn), d_prev=z(nn), gp=gp)
    cracked = (C.precrack_nodes_grid(case) if dp.mesh is None
               else C.precrack_nodes(case, dp.mesh))
    st.d[cracked] = 1.0
    st.d_prev[cracked] = 1.0
    return st


class _Single:
    """N = 1: one DeviceSession on the whole mesh, state built on the device."""

    def __init__(self, dp, case, local):
        from paper_2209_07969_b200 import configs as C
        from paper_2209_07969_b200.session import DeviceSession

        self.s = DeviceSession(dp.layout, dp.params, dp.config, device=local)
        self.dp = dp
        self.n_local = dp.layout.n_nodes
        segs, radius = C.precrack_segments(case)
        lay = dp.layout
        self.s.init_state(segs if len(segs) else None, radius, lay.nx * lay.hx, lay.ny * lay.hy)

    def step(self, scheme):
        return self.s.step(scheme, self.dp.bcs, self.dp.pins)


class _Strip:
    """N > 1: one row strip per rank, NCCL halos and all-reduces (pf_create_strip)."""

    def __init__(self, dp, case, rank, ws, local):
        import torch.distributed as dist

        from paper_2209_07969_b200.dist import StripSession, nccl_unique_id

        obj = [nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        self.s = StripSession(dp.layout, dp.params, dp.config, rank, ws, "nccl",
                              device=local, nccl_id=obj[0])
        self.dp = dp
        self.n_local = self.s.strip.n_local
        self.push(host_initial_state(dp, case, pinned=False))

    def push(self, state):
        g = state.gp
        self.s.push_global(state.u, state.d, state.d_prev, g.tr_eps_plus, g.dev_dot_dev,
                           g.psi_plus, g.psi_max)

    def step(self, scheme):
        return self.s.step(scheme, self.dp.bcs, self.dp.pins)


def dominant_kernel(sess, iters_d, iters_u):
    """The candidate kernels of the load step with their CUDA-event timing on the final state
    (pf_bench_mg_kernel) and their launches in the timed region: the fine-level marches of the two
    multigrid PCGs, each launched once per multigrid iteration of its solver."""
    kinds = sess.solver_kinds()
    out = []
    cands = []
    if kinds["phase_field"] == "multigrid_pcg":
        cands += [("k_mgs_fine_smooth", 11, iters_d), ("k_mgs_pcg", 12, iters_d),
                  ("k_mgs_fine_resid", 10, iters_d)]
    if kinds["momentum"] == "multigrid_pcg":
        cands += [("k_mg_pcg", 2, iters_u), ("k_mg_fine_smooth", 1, iters_u),
                  ("k_mg_fine_resid", 0, iters_u)]
    for name, code, launches in cands:
        ms, nbytes, desc = sess.bench_mg_kernel(code, 20)
        out.append({"kernel": name, "ms_per_launch": ms, "algorithmic_bytes": nbytes,
                    "bytes_note": desc, "achieved_gbs": nbytes / (ms * 1e-3) / 1e9,
                    "launches_in_timed_region": launches,
                    "ms_in_timed_region": ms * launches})
    return out


def run_ours(args, ws, rank, local):
    from paper_2209_07969_b200 import configs as C
    from paper_2209_07969_b200 import schemes
    from paper_2209_07969_b200.assembly import Discretization

    case = C.get_case(args.case)
    if ws > 1:
        import torch
        import torch.distributed as dist

        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dp = C.device_problem(case)
    n_nodes, n_elems = dp.layout.n_nodes, dp.layout.n_elems
    run = _Single(dp, case, local) if ws == 1 else _Strip(dp, case, rank, ws, local)
    sess = run.s if ws == 1 else run.s.sess
    l2 = sess.device_info()["l2_bytes"]
    flush = 200.0 * n_nodes < 4.0 * l2  # the PCG working set fits L2: flush between steps
    for _ in range(args.warmup):
        run.step(args.scheme)
    sess.synchronize()
    barrier(ws)
    tot = dict(ms=0.0, n_stag=0, cg_u=0, cg_d=0, ms_u=0.0, ms_d=0.0, dofit=0.0, launches=0,
               cgl_u=0, cgl_d=0, nr_u=0, nr_d=0)
    per_step = []
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            if flush:
                sess.flush_l2()
            barrier(ws)
            st = run.step(args.scheme)  # synchronizes at its end
            ms = st.step_ms  # CUDA events on the solver stream around the whole load step
            per_step.append(ms)
            tot["ms"] += ms
            tot["n_stag"] += st.n_stag
            tot["nr_u"] += st.n_nr_u
            tot["nr_d"] += st.n_nr_d
            tot["cg_u"] += st.cg_iters_u
            tot["cg_d"] += st.cg_iters_d
            tot["ms_u"] += st.kernel_ms_u
            tot["ms_d"] += st.kernel_ms_d
            tot["dofit"] += st.cg_dofiters_u + st.cg_dofiters_d
            tot["launches"] += st.launches
            tot["cgl_u"] += st.cg_launches_u
            tot["cgl_d"] += st.cg_launches_d
    sess.synchronize()
    barrier(ws)
    t_max = allreduce_max(ws, tot["ms"])
    kinds = sess.solver_kinds()
    mg = sess.mg_info()
    kernels = dominant_kernel(sess, tot["cg_d"], tot["cg_u"]) if ws == 1 else []
    if ws == 1:
        sess.close()
    # e2e: host SolverState in, host SolverState out, every step (copies inside the timing)
    e2e = None
    if ws > 1:  # scatter the host state to the strips, step, gather the owned results
        run2 = _Strip(dp, case, rank, ws, local)
        hst = host_initial_state(dp, case, pinned=False)
        for _ in range(args.warmup):
            run2.push(hst)
            run2.step(args.scheme)
            gather_full(run2.s.owned_state(), hst, ws)
        barrier(ws)
        e_stag = 0
        t0 = time.perf_counter()
        for _ in range(args.steps):
            run2.push(hst)
            s2 = run2.step(args.scheme)
            gather_full(run2.s.owned_state(), hst, ws)
            e_stag += s2.n_stag
        e_ms = allreduce_max(ws, (time.perf_counter() - t0) * 1e3)
        nl, el = run2.s.strip.n_local, run2.s.strip.layout.n_elems
        e2e = {"value": 3 * n_nodes * e_stag / (e_ms / 1e3), "unit": "DOF-iter/s",
               "h2d_bytes_per_step": 8 * (4 * nl + 16 * el),
               "d2h_bytes_per_step": 8 * (4 * nl + 16 * el), "ms_per_step": e_ms / args.steps,
               "path": "dist.StripSession: scatter host SolverState, step, gather owned "
                       "results, all-gather into every rank's host state"}
        run2.s.close()
    if ws == 1:
        disc = (Discretization.from_layout(dp.layout) if dp.mesh is None
                else Discretization(dp.mesh))
        kind = schemes.SchemeKind(args.scheme)

        def e2e_run(state, warm, steps):
            for _ in range(warm):
                schemes.staggered_step(disc, state, kind, dp.bcs, dp.params, dp.config, dp.pins)
            n_stag = 0
            t0 = time.perf_counter()
            for _ in range(steps):
                s2 = schemes.staggered_step(disc, state, kind, dp.bcs, dp.params, dp.config,
                                            dp.pins)
                n_stag += s2.n_stag
            return n_stag, (time.perf_counter() - t0) * 1e3

        h2d = 8 * (2 * n_nodes + 2 * n_nodes + 4 * n_elems)  # u, d, d_prev, gp.psi_max
        d2h = 8 * (4 * n_nodes + 4 * 4 * n_elems)  # u, d, d_prev, 4 GP arrays
        if schemes.SYNC_GP_STRAIN:
            d2h += 8 * (16 + 4) * n_elems  # gp.strain, gp.tr_eps
        pst = host_initial_state(dp, case, pinned=True)
        e_stag, e_ms = e2e_run(pst, args.warmup, args.steps)
        del pst
        pg = host_initial_state(dp, case, pinned=False)
        pg_steps = min(args.steps, 3)
        p_stag, p_ms = e2e_run(pg, 1, pg_steps)
        del pg
        for s in disc.__dict__.get("_pfb200_sessions", {}).values():
            s.close()
        e2e = {"value": 3 * n_nodes * e_stag / (e_ms / 1e3), "unit": "DOF-iter/s",
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
               "ms_per_step": e_ms / args.steps,
               "path": "paper_2209_07969_b200.schemes.staggered_step with a host SolverState "
                       "in page-locked arrays (load steps after the same W warm-up steps)",
               "pageable": {"value": 3 * n_nodes * p_stag / (p_ms / 1e3),
                            "ms_per_step": p_ms / pg_steps, "steps": pg_steps,
                            "note": "reference-style SolverState of ordinary numpy arrays "
                                    "(staged copies); 1 untimed warm-up step"}}
    ndof = 3 * n_nodes
    value = ndof * tot["n_stag"] / (t_max / 1e3)
    peak, peak_src = peaks()
    roofline = None
    if kernels:
        dom = max(kernels, key=lambda k: k["ms_in_timed_region"])
        traffic = None
        tpath = os.path.join(ROOT, "profiles", "r2_kernel_traffic.json")
        if os.path.exists(tpath):
            with open(tpath) as f:
                tj = json.load(f)
            ent = tj.get(dom["kernel"])
            if ent and ent.get("case") == args.case:
                traffic = ent["dram_bytes_per_launch"]
        roofline = {"kernel": dom["kernel"], "bound": "hbm", "achieved": dom["achieved_gbs"],
                    "peak": peak, "unit": "GB/s", "frac": dom["achieved_gbs"] / peak,
                    "traffic": traffic, "peak_source": peak_src,
                    "algorithmic_bytes_per_launch": dom["algorithmic_bytes"],
                    "algorithmic_bytes": dom["bytes_note"],
                    "ms_per_launch": dom["ms_per_launch"],
                    "share_of_timed_region": dom["ms_in_timed_region"] / t_max,
                    "timing": "CUDA events on the solver stream, 20 re-launches on the final "
                              "state after the timed region (pf_bench_mg_kernel)",
                    "candidates": kernels}
    launches = int(allreduce_sum(ws, float(tot["launches"])))
    res = {
        "metric": METRIC,
        "value": value,
        "unit": "DOF-iter/s",
        "n_gpus": ws,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": t_max / args.steps,
        "higher_is_better": True,
        "scaling": "weak" if ws == 1 else "strong",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (BASELINE recipe: seeded structured mesh and pre-cracks, no dataset)",
        "config": {
            "workload": f"{args.case}: {case.note}; scheme {args.scheme}; load steps "
                        f"{args.warmup + 1}..{args.warmup + args.steps}",
            "n_nodes": n_nodes, "n_elems": n_elems, "dofs": ndof,
            "parallelism": "single-gpu" if ws == 1 else f"row strips x{ws} (NCCL halos)",
            "l2": ("flushed (256 MiB write) before each timed load step" if flush else
                   "inputs larger than L2 (working set ~25 GB vs 126 MB L2): no flush"),
            "timing": "CUDA events on the solver stream around each pf_staggered_step; "
                      "max over ranks",
        },
        "load_steps_per_s": args.steps / (t_max / 1e3),
        "solver_dof_iter_per_s": allreduce_sum(ws, tot["dofit"]) / (t_max / 1e3),
        "n_stag_total": tot["n_stag"],
        "newton": {"momentum": tot["nr_u"], "phase_field": tot["nr_d"]},
        "solvers": kinds,
        "pcg_iters": {"momentum": tot["cg_u"], "phase_field": tot["cg_d"],
                      "momentum_solves": tot["cgl_u"], "phase_field_solves": tot["cgl_d"]},
        "kernel_ms": {"momentum_pcg": tot["ms_u"], "phase_field_pcg": tot["ms_d"]},
        "roofline": roofline,
        "momentum_solver": ({"kind": "multigrid PCG (Galerkin V(1,1), CUDA graph)",
                             "levels": mg["n_levels"], "hierarchy_builds": mg.get("setups"),
                             "us_per_iteration": 1e3 * tot["ms_u"] / max(tot["cg_u"], 1)}
                            if mg["n_levels"] else {"kind": "Jacobi PCG"}),
        "e2e": e2e,
        "gpu_launches": launches,
        "clocks": clk.summary(),
        "per_step_ms": [round(x, 3) for x in per_step],
    }
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        res["cpu_baseline"] = cpu_baseline()
    if ws > 1:
        run.s.close()
        import torch.distributed as dist

        dist.destroy_process_group()
    return res if rank == 0 else None


def gather_full(own, state, ws):
    """All-gather the ranks' owned nodal / cell results into the full host SolverState."""
    import torch
    import torch.distributed as dist

    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"

    def allgather_rows(mat):
        t = torch.from_numpy(np.ascontiguousarray(mat)).to(dev)
        n = torch.tensor([t.shape[0]], device=dev)
        ns = [torch.zeros_like(n) for _ in range(ws)]
        dist.all_gather(ns, n)
        m = int(max(int(x) for x in ns))
        pad = torch.zeros((m, t.shape[1]), dtype=t.dtype, device=dev)
        pad[: t.shape[0]] = t
        outs = [torch.empty_like(pad) for _ in range(ws)]
        dist.all_gather(outs, pad)
        return np.concatenate([o[: int(k)].cpu().numpy() for o, k in zip(outs, ns)])

    nodes = allgather_rows(np.column_stack([own["nodes"].astype(np.float64), own["u"],
                                            own["d"], own["d_prev"]]))
    ids = nodes[:, 0].astype(np.int64)
    state.u.reshape(-1, 2)[ids] = nodes[:, 1:3]
    state.d[ids] = nodes[:, 3]
    state.d_prev[ids] = nodes[:, 4]
    gp = state.gp
    cells = allgather_rows(np.column_stack([own["cells"].astype(np.float64)] + [
        own[k].reshape(-1, 4) for k in ("tr_eps_plus", "dev_dot_dev", "psi_plus", "psi_max")]))
    cid = cells[:, 0].astype(np.int64)
    for j, k in enumerate(("tr_eps_plus", "dev_dot_dev", "psi_plus", "psi_max")):
        getattr(gp, k)[cid] = cells[:, 1 + 4 * j: 5 + 4 * j]


def barrier(ws):
    if ws > 1:
        import torch.distributed as dist

        dist.barrier()


def allreduce_sum(ws, v):
    if ws == 1:
        return v
    import torch
    import torch.distributed as dist

    t = torch.tensor([v], dtype=torch.float64, device="cuda")
    dist.all_reduce(t)
    return float(t.item())


def allreduce_max(ws, v):
    if ws == 1:
        return v
    import torch
    import torch.distributed as dist

    t = torch.tensor([v], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# -------------------------------------------------------------------------------------------
def oracle_window(case_name, scheme, warmup, max_steps, budget_s):
    """The CPU oracle port: `warmup` untimed load steps from step 1, then timed load steps
    until max_steps or the time budget."""
    from oracle.phasefield_oracle import oracle_api
    from paper_2209_07969_b200 import configs as C

    case = C.get_case(case_name)
    pb = C.setup(case, oracle_api())

    def one():
        return pb.api.staggered_step(pb.disc, pb.state, scheme, pb.bcs, pb.params, pb.config,
                                     pb.pins)

    for _ in range(warmup):
        one()
    n_stag, wall, steps = 0, 0.0, 0
    while steps < max_steps and (steps == 0 or wall < budget_s):
        t0 = time.perf_counter()
        st = one()
        wall += time.perf_counter() - t0
        n_stag += st.n_stag
        steps += 1
    ndof = 3 * pb.mesh.n_nodes
    return ndof * n_stag / wall, steps, n_stag, wall


def cpu_baseline():
    v, steps, n_stag, wall = oracle_window("cfg2", "S1", 0, 1, 0.0)
    return {"value": v, "unit": "DOF-iter/s", "cores": 1, "kind": "port",
            "sample": f"oracle port (SuperLU direct solves, like the reference default) on load "
                      f"step 1 of cfg2 (512^2, 790 k DOFs; {n_stag} staggered iteration(s), "
                      f"{wall:.1f} s): config 5 itself cannot be set up on a CPU (the "
                      f"reference's Discretization needs ~120 GB and a 201 M-DOF SuperLU "
                      f"factorisation is infeasible, SURVEY.md §5)"}


def run_reference(args, ws, rank):
    if rank != 0:
        return None
    from paper_2209_07969_b200 import configs as C

    case = C.get_case(args.case)
    cores = os.cpu_count() or 1
    budget = float(os.environ.get("PFB200_REF_BUDGET_S", "120"))
    sec_case = "cfg2"
    v, steps, n_stag, wall = oracle_window(sec_case, args.scheme, args.warmup, args.steps, budget)
    sample = (f"CPU oracle port of the reference algorithm (SuperLU direct solves; SuperLU is "
              f"single-threaded, numpy may use {cores} threads) on {sec_case}: load steps "
              f"1..{args.warmup} untimed, steps {args.warmup + 1}..{args.warmup + steps} timed "
              f"({n_stag} staggered iterations, {wall:.1f} s; {budget:.0f} s budget)")
    runnable = args.case not in ("cfg5",)
    line = {
        "impl": "reference",
        "metric": METRIC,
        "value": v if not runnable or args.case == sec_case else None,
        "unit": "DOF-iter/s", "n_gpus": ws, "steps": steps,
        "requested_steps": args.steps, "warmup": args.warmup,
        "ms_per_step": wall * 1e3 / steps if steps else None,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (BASELINE recipe)",
        "config": {"workload": f"{args.case}: {case.note}; scheme {args.scheme}"},
        "cpu_baseline": {"value": v, "unit": "DOF-iter/s", "cores": cores, "kind": "port",
                         "sample": sample},
        "e2e": {"value": v, "unit": "DOF-iter/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    if args.case != sec_case:
        line["value"] = None
        line["e2e"]["value"] = None
        line["unavailable_reason"] = (
            f"{args.case} is not runnable by the reference's CPU algorithm (SURVEY.md §8(d): the "
            f"reference's Discretization needs ~120 GB and each Newton step a 201 M-DOF SuperLU "
            f"factorisation); the secondary line times the same algorithm on cfg2")
        line["secondary"] = {"case": sec_case, "value": v, "unit": "DOF-iter/s",
                             "warmup": args.warmup, "steps": steps, "sample": sample}
    return line


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--case", default="cfg5")
    ap.add_argument("--scheme", default="S1")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        print("note: warmup < 3 violates the timing rules", file=sys.stderr)
    ws, rank, local = dist_env()
    res = run_reference(args, ws, rank) if args.impl == "reference" else run_ours(
        args, ws, rank, local)
    if rank == 0 and res is not None:
        print(json.dumps(res))


if __name__ == "__main__":
    main()
