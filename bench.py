"""Benchmark: load steps of BASELINE configs[1] (512x512 notched tension, 790k DOFs, FP64).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--case cfg2] [--scheme S1]

A "step" is one load step (``staggered_step``, reference schemes.py:332-392) of the case's own
schedule: W untimed warm-up load steps advance the state, then K load steps are timed.

* ``value``   — DOF-iterations/s (SURVEY.md §8(d) reading 1a: 3*N_nodes * sum n_stag / time),
  device-resident state, CUDA events on the solver stream around each load step, L2 flushed
  (256 MiB write) before every timed step, outside the timed region.
* ``e2e``     — the same metric through the reference-facing drop-in
  ``paper_2209_07969_b200.schemes.staggered_step`` with the caller's HOST SolverState: every
  step uploads the state, solves, and downloads the state (all copies inside the timed region).
* ``roofline``— the dominant single kernel: with the multigrid momentum solver (default) the
  phase-field PCG (``k_cg_st`` on the assembled stencil for L2-resident meshes, else
  ``k_cg_sr<false>``; algorithmic bytes 72 B * N_nodes + 32 B * N_cells per PCG iteration,
  SURVEY.md §8(d)); with PFB200_MG=0 the momentum PCG (168 B * N_nodes) / its CUDA-event time.
  ``momentum_solver`` summarises the multigrid PCG graph.
* ``cpu_baseline`` — the CPU oracle port (oracle/phasefield_oracle.py, SuperLU like the
  reference default) on the first load step of the same case, rank 0 only.
* ``--gpus N`` (torchrun, one process per GPU) — the same cfg2 problem split into N row strips
  (``dist.StripSession``: NCCL halo rows + all-reduces captured in CUDA graphs), strong
  scaling; value = global DOF-iterations / max-over-ranks device time.
* ``--impl reference`` — the reference's CPU algorithm (the oracle port; the Python reference
  does not travel to the GPU box) on the same case/metric; load steps until K are done or a
  time budget is spent.
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

MOM_BYTES_PER_NODE = 168.0          # momentum PCG iteration
EVO_BYTES_PER_NODE, EVO_BYTES_PER_ELEM = 72.0, 32.0


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
    thread (the timed region lasts ~70 ms, too short for nvidia-smi's 100+ ms start-up and
    200 ms interval); `nvidia-smi -lms 200` when NVML is not importable."""

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
class _Single:
    """N = 1: one DeviceSession on the whole mesh (persistent cooperative PCG)."""

    def __init__(self, pb, local):
        from paper_2209_07969_b200.session import DeviceSession

        self.s = DeviceSession(pb.disc.layout, pb.params, pb.config, device=local)
        self.pb = pb
        self.n_local = pb.mesh.n_nodes

    def push(self, state):
        self.s.push_state(state)

    def step(self, scheme):
        return self.s.step(scheme, self.pb.bcs, self.pb.pins)


class _Strip:
    """N > 1: one row strip per rank, NCCL halos and all-reduces (pf_create_strip)."""

    def __init__(self, pb, rank, ws, local):
        import torch.distributed as dist

        from paper_2209_07969_b200.dist import StripSession, nccl_unique_id

        obj = [nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        self.s = StripSession(pb.disc.layout, pb.params, pb.config, rank, ws, "nccl",
                              device=local, nccl_id=obj[0])
        self.pb = pb
        self.n_local = self.s.strip.n_local

    def push(self, state):
        g = state.gp
        self.s.push_global(state.u, state.d, state.d_prev, g.tr_eps_plus, g.dev_dot_dev,
                           g.psi_plus, g.psi_max)

    def step(self, scheme):
        return self.s.step(scheme, self.pb.bcs, self.pb.pins)


def run_ours(args, ws, rank, local):
    from paper_2209_07969_b200 import configs as C
    from paper_2209_07969_b200 import schemes

    case = C.get_case(args.case)
    if ws > 1:
        import torch
        import torch.distributed as dist

        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    pb = C.setup(case, C.b200_api())
    n_nodes, n_elems = pb.mesh.n_nodes, pb.mesh.n_elems
    run = _Single(pb, local) if ws == 1 else _Strip(pb, rank, ws, local)
    sess = run.s if ws == 1 else run.s.sess
    run.push(pb.state)
    for _ in range(args.warmup):
        run.step(args.scheme)
    sess.synchronize()
    barrier(ws)
    tot = dict(ms=0.0, n_stag=0, cg_u=0, cg_d=0, ms_u=0.0, ms_d=0.0, dofit=0.0, launches=0,
               cgl_u=0, cgl_d=0)
    per_step = []
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            sess.flush_l2()  # inputs of a 512^2 load step fit in L2: flush between steps
            barrier(ws)
            st = run.step(args.scheme)  # synchronizes at its end
            ms = st.step_ms  # CUDA events on the solver stream around the whole load step
            per_step.append(ms)
            tot["ms"] += ms
            tot["n_stag"] += st.n_stag
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
    # e2e: host SolverState in, host SolverState out, every step (copies inside the timing)
    pb2 = C.setup(case, C.b200_api())
    kind = schemes.SchemeKind(args.scheme)
    e2e_stag = 0
    if ws == 1:
        for _ in range(args.warmup):
            schemes.staggered_step(pb2.disc, pb2.state, kind, pb2.bcs, pb2.params, pb2.config,
                                   pb2.pins)
        t0 = time.perf_counter()
        for _ in range(args.steps):
            s2 = schemes.staggered_step(pb2.disc, pb2.state, kind, pb2.bcs, pb2.params,
                                        pb2.config, pb2.pins)
            e2e_stag += s2.n_stag
        e2e_ms = (time.perf_counter() - t0) * 1e3
        h2d = 8 * (2 * n_nodes + 2 * n_nodes + 4 * n_elems)  # u, d, d_prev, gp.psi_max
        d2h = 8 * (4 * n_nodes + 4 * 4 * n_elems)  # u, d, d_prev, 4 GP arrays
        if schemes.SYNC_GP_STRAIN:
            d2h += 8 * (16 + 4) * n_elems  # gp.strain, gp.tr_eps
        e2e_path = "paper_2209_07969_b200.schemes.staggered_step with host SolverState"
    else:
        run2 = _Strip(pb2, rank, ws, local)
        ss = run2.s
        for _ in range(args.warmup):
            run2.push(pb2.state)
            run2.step(args.scheme)
        barrier(ws)
        t0 = time.perf_counter()
        for _ in range(args.steps):
            run2.push(pb2.state)  # scatter the host state to the strip
            s2 = run2.step(args.scheme)
            gather_full(ss.owned_state(), pb2.state, ws)  # owned results -> every host copy
            e2e_stag += s2.n_stag
        e2e_ms = allreduce_max(ws, (time.perf_counter() - t0) * 1e3)
        nl, el = ss.strip.n_local, ss.strip.layout.n_elems
        h2d = 8 * (4 * nl + 16 * el)
        d2h = 8 * (4 * nl + 16 * el)
        e2e_path = ("dist.StripSession: scatter host SolverState, step, gather owned results, "
                    "all-gather into every rank's host state")
        run2.s.close()
    ndof = 3 * n_nodes
    value = ndof * tot["n_stag"] / (t_max / 1e3)
    peak, peak_src = peaks()
    n_cg = run.n_local
    mom_bytes = MOM_BYTES_PER_NODE * n_cg
    evo_bytes = EVO_BYTES_PER_NODE * n_cg + EVO_BYTES_PER_ELEM * n_elems / ws
    evo_achieved = (tot["cg_d"] * evo_bytes / 1e9) / (tot["ms_d"] / 1e3) if tot["ms_d"] else 0.0
    mg = sess.mg_info() if ws == 1 else {"n_levels": 0}
    if mg["n_levels"]:
        # The momentum solves run as the multigrid PCG graph (~30 small kernels per iteration,
        # no single dominant kernel); the largest single kernel is the phase-field Jacobi PCG
        # (k_cg<false, *>, one persistent launch per solve): its roofline is reported.
        kinds = sess.solver_kinds()
        if kinds["phase_field"] == "stencil_pcg":
            rl_kernel = ("k_cg_st (phase-field single-reduction Jacobi PCG on the assembled "
                         "stencil, persistent cooperative; solves without the SPD probe)")
            tkey = "k_cg_st"
        else:
            rl_kernel = ("k_cg_sr<false> (phase-field single-reduction Jacobi PCG, persistent "
                         "cooperative; solves without the SPD probe)")
            tkey = "k_cg_evo"
        achieved, rl_bytes = evo_achieved, "72 B x N_nodes + 32 B x N_cells per phase-field PCG iteration"
        iters_key, launches_key = "cg_d", "cgl_d"
    else:
        rl_kernel = ("k_cg<true, *> (momentum PCG, persistent cooperative)" if ws == 1 else
                     "momentum PCG (k_cg_a/k_cg_b + NCCL, rank 0's strip)")
        achieved = (tot["cg_u"] * mom_bytes / 1e9) / (tot["ms_u"] / 1e3) if tot["ms_u"] else 0.0
        rl_bytes = "168 B x N_nodes per momentum PCG iteration"
        tkey, iters_key, launches_key = "k_cg", "cg_u", "cgl_u"
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "k_cg_traffic.json")
    if os.path.exists(tpath) and ws == 1:
        with open(tpath) as f:
            tj = json.load(f)
        ent = tj.get(tkey)
        if ent and ent.get("case") == args.case and tot[launches_key]:
            if "dram_bytes_per_launch" in ent:
                traffic = ent["dram_bytes_per_launch"]
            else:
                traffic = ent["dram_bytes_per_iter"] * tot[iters_key] / tot[launches_key]
    launches = int(allreduce_sum(ws, float(tot["launches"])))
    res = {
        "metric": "DOF-iterations/s of staggered solve (FP64)",
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
        "data": "synthetic (BASELINE configs[1] recipe: seeded structured mesh, no dataset)",
        "config": {
            "workload": f"{args.case}: {case.note}; scheme {args.scheme}; load steps "
                        f"{args.warmup + 1}..{args.warmup + args.steps}",
            "n_nodes": n_nodes, "n_elems": n_elems, "dofs": ndof,
            "parallelism": "single-gpu" if ws == 1 else f"row strips x{ws} (NCCL halos)",
            "l2": "flushed (256 MiB write) before each timed load step, outside the timing",
            "timing": "CUDA events on the solver stream around each pf_staggered_step; "
                      "max over ranks",
        },
        "load_steps_per_s": args.steps / (t_max / 1e3),
        "solver_dof_iter_per_s": allreduce_sum(ws, tot["dofit"]) / (t_max / 1e3),
        "n_stag_total": tot["n_stag"],
        "pcg_iters": {"momentum": tot["cg_u"], "phase_field": tot["cg_d"],
                      "momentum_launches": tot["cgl_u"], "phase_field_launches": tot["cgl_d"]},
        "kernel_ms": {"momentum_pcg": tot["ms_u"], "phase_field_pcg": tot["ms_d"]},
        "roofline": {
            "kernel": rl_kernel,
            "bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
            "frac": achieved / peak, "traffic": traffic,
            "peak_source": peak_src,
            "algorithmic_bytes": rl_bytes,
            "note": "cfg2's PCG working set (~50 MB) is L2-resident: the fraction mixes L2 and "
                    "HBM traffic (SURVEY.md 8(d)); cfg3-5 are the HBM-bound sizes.  k_cg_st "
                    "moves more than the algorithmic bytes (assembled rows 80 B + neighbour "
                    "ids 40 B per node instead of 32 B per cell): achieved counts only the "
                    "algorithmic bytes",
        },
        "momentum_solver": ({"kind": "multigrid PCG (Galerkin V(1,1), CUDA graph)",
                             "precision": "FP64 operator, residuals, dot products and stopping "
                                          "test; grid-level coarse stencils stored FP32 "
                                          "(preconditioner only)",
                             "levels": mg["n_levels"], "hierarchy_builds": mg.get("setups"),
                             "iterations": tot["cg_u"], "solves": tot["cgl_u"],
                             "us_per_iteration": 1e3 * tot["ms_u"] / max(tot["cg_u"], 1)}
                            if mg["n_levels"] else {"kind": "Jacobi PCG"}),
        "e2e": {"value": ndof * e2e_stag / (e2e_ms / 1e3), "unit": "DOF-iter/s",
                "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "ms_per_step": e2e_ms / args.steps, "path": e2e_path},
        "gpu_launches": launches,
        "clocks": clk.summary(),
        "per_step_ms": [round(x, 3) for x in per_step],
    }
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        res["cpu_baseline"] = cpu_baseline(args, case)
    if ws > 1:
        run.s.close()
        import torch.distributed as dist

        dist.destroy_process_group()
    else:
        sess.close()
    return res if rank == 0 else None


def barrier(ws):
    if ws > 1:
        import torch.distributed as dist

        dist.barrier()


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
def oracle_steps(case_name, scheme, max_steps, budget_s):
    """Run the CPU oracle port from load step 1 until max_steps or the time budget."""
    from oracle.phasefield_oracle import oracle_api
    from paper_2209_07969_b200 import configs as C

    case = C.get_case(case_name)
    pb = C.setup(case, oracle_api())
    n_stag, wall, steps = 0, 0.0, 0
    while steps < max_steps and (steps == 0 or wall < budget_s):
        t0 = time.perf_counter()
        st = pb.api.staggered_step(pb.disc, pb.state, scheme, pb.bcs, pb.params, pb.config,
                                   pb.pins)
        wall += time.perf_counter() - t0
        n_stag += st.n_stag
        steps += 1
    ndof = 3 * pb.mesh.n_nodes
    return ndof * n_stag / wall, steps, n_stag, wall


def cpu_baseline(args, case):
    v, steps, n_stag, wall = oracle_steps(args.case, args.scheme, 1, 0.0)
    return {"value": v, "unit": "DOF-iter/s", "cores": 1, "kind": "port",
            "sample": f"oracle port (SuperLU, like the reference default) on load step 1 of "
                      f"{args.case} ({n_stag} staggered iteration(s), {wall:.1f} s)"}


def run_reference(args, ws, rank):
    if rank != 0:
        return None
    budget = float(os.environ.get("PFB200_REF_BUDGET_S", "150"))
    v, steps, n_stag, wall = oracle_steps(args.case, args.scheme, args.steps, budget)
    from paper_2209_07969_b200 import configs as C

    case = C.get_case(args.case)
    cores = os.cpu_count() or 1
    sample = (f"CPU oracle port of the reference algorithm (SuperLU direct solves; SuperLU is "
              f"single-threaded, numpy may use {cores} threads) on load steps 1..{steps} of "
              f"{args.case} ({n_stag} staggered iterations, {wall:.1f} s); warm-up steps "
              f"skipped and steps capped by a {budget:.0f} s budget")
    return {
        "impl": "reference",
        "metric": "DOF-iterations/s of staggered solve (FP64)",
        "value": v, "unit": "DOF-iter/s", "n_gpus": ws, "steps": steps,
        "requested_steps": args.steps, "warmup": 0, "ms_per_step": wall * 1e3 / steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (BASELINE configs[1] recipe)",
        "config": {"workload": f"{args.case}: {case.note}; scheme {args.scheme}"},
        "cpu_baseline": {"value": v, "unit": "DOF-iter/s", "cores": cores, "kind": "port",
                         "sample": sample},
        "e2e": {"value": v, "unit": "DOF-iter/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--case", default="cfg2")
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
