#!/usr/bin/env python
"""bench.py -- zone-cycles/s of the fp64 SALE cycle (arXiv 2209.01983) on B200.

A "step" is one SALE cycle (every §8(a) row: Lagrangian phase S1-S7, Eulerian
remap R1-R5 in EULER mode, halo exchange X1, dt min-reduction X2) over the
whole mesh.  Default workload: BASELINE.json config 4 ("C4": Sedov-Taylor 3D,
256^3 cells per GPU, Eulerian rezoning, fp64, z-slabs over the GPUs -> weak
scaling); --config C3 selects the strong-scaling Lagrangian 320^3 mesh.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C4|C3]
    python bench.py --impl reference ...   # the CPU oracle arm (rank 0 only)

One JSON line on rank 0.  Timing: W untimed cycles, then K cycles bracketed by
barrier + cuda.synchronize on both sides, CUDA events on the launching stream,
max over ranks.  Inputs (the mesh state, >= 1.1 GB per GPU) are larger than L2.
"""
from __future__ import annotations

import argparse
import csv
import io
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_2209_01983_b200 import configs  # noqa: E402

METRIC = "zone-cycles/s (fp64 SALE cycle)"
UNIT = "zone-cycles/s"
# algorithmic bytes per zone-cycle (state read + written once, fp64)
ALGO_BYTES = {configs.LAGRANGE: 120.0, configs.EULER: 80.0}
# algorithmic FP64-pipe instructions per zone-cycle of each kernel
# class (faces / edges / nodes computed once; a quantity two kernels both evaluate
# -- the t^n areas, corner vectors, hourglass modes and corner forces the energy
# kernel re-forms -- counted once; an IEEE fp64 div or sqrt = 8 FP64 instructions,
# its fast-path SASS sequence).  Lagrange: state 390 + force 405 + energy 230;
# Euler: state 138 + force 276 + energy 236 (the target geometry is tabled), remap
# R1-R4 406.
ALGO_FP64 = {configs.LAGRANGE: {"lagrange": 1025.0, "remap": 0.0},
             configs.EULER: {"lagrange": 650.0, "remap": 406.0}}
# kernel name prefixes of each timing class (for the ncu traffic file)
CLASS_KERNELS = {"lagrange": ("kc_", "ke_state", "kl_state"), "remap": ("kr_", "kn_update", "k_mat_flux")}
REASON_BITS = {"hw_slowdown": "hw_slowdown", "hw_thermal_slowdown": "hw_thermal_slowdown",
               "sw_thermal_slowdown": "sw_thermal_slowdown", "sw_power_cap": "sw_power_cap"}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def traffic(config_name: str, dom: str):
    """DRAM bytes (read + write) per launch group of the dominant kernel class, and the
    class's time-weighted FP64-pipe utilisation, from the committed ncu --set full
    capture of this workload (profiles/traffic_<cfg>.json, written by
    scripts/traffic_from_ncu.py); Nones if absent."""
    try:
        with open(os.path.join(ROOT, "profiles", f"traffic_{config_name}.json")) as f:
            d = json.load(f)
        per = d["dram_bytes_per_launch"]
        ks = [k for k in per if k.startswith(CLASS_KERNELS[dom])]
        tot = sum(per[k] for k in ks)
        fp = d.get("fp64_pipe_pct_of_active")
        pipe = None
        if fp:
            t = d["gpu_time_ns_per_launch"]
            pipe = sum(fp[k] * t[k] for k in ks) / sum(t[k] for k in ks)
        return (tot if tot > 0 else None), d.get("source"), pipe
    except Exception:
        return None, None, None


def fp64_peak():
    """FP64-pipe instruction rate (T thread-instr/s): the DADD chain rate measured on
    this pool's B200 by tools/fp64_peak.cu (profiles/r01_fp64_peak.json); fallback
    derived from unit counts: 148 SM x 64 FP64 lanes x 1.965 GHz = 18.6 T/s."""
    try:
        with open(os.path.join(ROOT, "profiles", "r01_fp64_peak.json")) as f:
            rows = [json.loads(x) for x in f if x.strip()]
        v = max(r["thread_inst_per_s_T"] for r in rows)
        return v, "measured (tools/fp64_peak.cu DADD chains, profiles/r01_fp64_peak.json)"
    except Exception:
        return 148 * 64 * 1.965e9 / 1e12, "derived (148 SM x 64 FP64 lanes x 1.965 GHz)"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.path = None

    def start(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}", "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        rows = []
        with open(self.path) as f:
            for r in csv.reader(f):
                if len(r) >= 9:
                    rows.append([x.strip() for x in r])
        os.unlink(self.path)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        reasons = set()
        for r in rows:
            for name, col in (("hw_slowdown", 5), ("hw_thermal_slowdown", 6),
                              ("sw_thermal_slowdown", 7), ("sw_power_cap", 8)):
                if r[col].lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(rows)}


def cpu_model() -> str:
    """The host CPU's model name (core count plus the lscpu model)."""
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def oracle_rate(cfg_sample: dict, seconds: float, min_cycles: int = 3, warm: int = 1):
    """Time the CPU oracle (as it stands, single thread) on a bounded sample."""
    import oracle as O
    o = O.Oracle(cfg_sample)
    if warm:
        o.step(warm)
    cells = cfg_sample["nx"] * cfg_sample["ny"] * cfg_sample["nz"]
    n, t0 = 0, time.perf_counter()
    while n < min_cycles or time.perf_counter() - t0 < seconds:
        rc, d = o.step(1)
        if rc:
            raise RuntimeError(f"oracle rc={rc}")
        n += 1
    dt = time.perf_counter() - t0
    return cells * n / dt, n, dt


def oracle_allcore(name: str, seconds: float):
    """All-core aggregate of the CPU oracle: one independent
    single-threaded oracle process per available core on the same bounded sample,
    run concurrently; the sum of their zone-cycles/s (replica throughput)."""
    ncore = len(os.sched_getaffinity(0))
    code = ("import json,sys; sys.path.insert(0, %r); import bench; "
            "s, _ = bench.sample_cfg(%r); v, n, dt = bench.oracle_rate(s, %r); print(json.dumps(v))"
            % (ROOT, name, seconds))
    procs = [subprocess.Popen([sys.executable, "-c", code], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL,
                              text=True) for _ in range(ncore)]
    rates = []
    for pr in procs:
        out, _ = pr.communicate()
        try:
            rates.append(float(out.strip().splitlines()[-1]))
        except Exception:
            pass
    return sum(rates), len(rates), ncore


def sample_cfg(name: str):
    """A bounded slab of the workload with the same cell size and physics."""
    cfg, _ = configs.config(name, 1)
    nzs = 4
    s = dict(cfg, nz=nzs, lz=cfg["lz"] * nzs / cfg["nz"])
    return s, f"{s['nx']}x{s['ny']}x{nzs} cells of {name} (same h, physics, mode), Sedov initial state"


def run_reference(args, world, rank):
    if rank != 0:
        return
    s, desc = sample_cfg(args.config)
    import oracle as O
    O.build()
    o = O.Oracle(s)
    o.step(args.warmup)
    cells = s["nx"] * s["ny"] * s["nz"]
    t0 = time.perf_counter()
    rc, done = o.step(args.steps)
    dt = time.perf_counter() - t0
    if rc or done != args.steps:
        raise RuntimeError(f"oracle rc={rc} done={done}")
    v = cells * args.steps / dt
    cfg, _ = configs.config(args.config, world)
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * dt / args.steps,
        "higher_is_better": True, "scaling": "weak" if args.config == "C4" else "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": workload_name(args.config), "sample": desc},
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": 1, "kind": "oracle", "sample": desc,
                         "cpu_model": cpu_model()},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


def workload_name(name):
    return {"C3": "C3: Sedov-Taylor 3D 320^3 cells, Lagrangian, fp64, strong scaling",
            "C4": "C4: Sedov-Taylor 3D 256^3 cells per GPU, Eulerian rezoning, fp64, weak scaling",
            }.get(name, name)


def totals(ctx):
    """Mass and total energy IE + KE (math.fsum, c.7) of the state, read back on the host."""
    import math
    M = ctx.get("NODE_MASS")
    ke = math.fsum((0.5 * M * (ctx.get("UX") ** 2 + ctx.get("UY") ** 2 + ctx.get("UZ") ** 2)).ravel())
    m = ctx.get("MASS")
    return math.fsum(m.ravel()), math.fsum((m * ctx.get("E")).ravel()) + ke


def time_cycles(ctx, cfg, steps, warmup, world, local, barrier, max_over_ranks, S, conservation=False):
    """W untimed cycles, then K cycles bracketed by barrier + synchronize, CUDA events
    on the context's stream, kernel-class timing and nvidia-smi clocks (max over ranks).
    conservation: also the relative change of mass and of IE + KE over the K cycles
    (read outside the timed region)."""
    import torch
    stream = ctx.stream
    rc, done = ctx.step(warmup)
    if rc or done != warmup:
        raise RuntimeError(f"warmup failed rc={rc} done={done}: {ctx.last_error()}")
    before = totals(ctx) if conservation else None
    sampler = ClockSampler(local)
    barrier()
    torch.cuda.synchronize()
    sampler.start()
    time.sleep(0.2)
    launches0 = ctx.launches()
    ctx.profile(True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    ctx.step_async(steps)
    e1.record(stream)
    torch.cuda.synchronize()
    rc, done = ctx.sync()
    barrier()
    clocks = sampler.stop()
    if rc or done != steps:
        raise RuntimeError(f"timed run failed rc={rc} done={done}: {ctx.last_error()}")
    ms = max_over_ranks(e0.elapsed_time(e1))
    launches = ctx.launches() - launches0
    prof = ctx.profile_read()
    ctx.profile(False)
    gcells = cfg["nx"] * cfg["ny"] * cfg["nz"]
    out = {"ms": ms, "launches": launches, "prof": prof, "clocks": clocks, "value": gcells * steps / (ms * 1e-3)}
    if conservation:
        after = totals(ctx)
        out["conservation"] = {
            "mass_rel_change": abs(after[0] - before[0]) / before[0],
            "energy_rel_change": abs(after[1] - before[1]) / before[1],
            "what": "over the timed cycles; mass exact up to round-off in both modes; IE + KE conserved to "
                    "round-off in Lagrange mode (compatible scheme with HG), not in Euler mode (the momentum "
                    "remap dissipates kinetic energy, reading Q17)"}
    return out


def roofline_of(config_name, mode, prof, ms, steps, local_cells):
    """The SALE kernels are bound by the FP64 pipe: the roofline ("alu")
    of the dominant kernel class; the HBM view rides along."""
    peak, peak_src = peaks()
    fpk, fpk_src = fp64_peak()
    dom = max(("lagrange", "remap"), key=lambda k: prof[k][0])
    dom_ms, dom_n = prof[dom]
    per_cycle_ms = dom_ms / steps                                  # the class may launch >1 group per cycle
    fp64_per_cycle = ALGO_FP64[mode][dom] * local_cells            # FP64 instr of the class per cycle
    achieved_t = fp64_per_cycle / (per_cycle_ms * 1e-3) / 1e12     # T instr/s
    cyc_fp64 = sum(ALGO_FP64[mode].values()) * local_cells
    cyc_t = cyc_fp64 / (ms / steps * 1e-3) / 1e12
    cyc_bytes = ALGO_BYTES[mode] * local_cells
    cycle_gbs = cyc_bytes / (ms / steps * 1e-3) / 1e9
    tr_bytes, tr_src, pipe = traffic(config_name, dom)
    return {"bound": "alu", "achieved": achieved_t, "peak": fpk, "unit": "T fp64-instr/s",
            "frac": achieved_t / fpk, "traffic": tr_bytes, "traffic_unit": "DRAM bytes per cycle of the class",
            "traffic_source": tr_src, "algo_bytes_per_cycle": ALGO_BYTES[mode] * local_cells,
            "traffic_bytes_per_zone": (tr_bytes / local_cells) if tr_bytes else None,
            "ncu_fp64_pipe_pct": pipe,
            "kernel": dom, "kernel_launch_groups_per_cycle": dom_n / steps,
            "kernel_ms_per_cycle": per_cycle_ms, "kernel_share_of_step": dom_ms / ms,
            "algo_fp64_instr_per_zone": ALGO_FP64[mode][dom], "peak_source": fpk_src,
            "whole_cycle": {"achieved": cyc_t, "frac": cyc_t / fpk,
                            "algo_fp64_instr_per_zone": sum(ALGO_FP64[mode].values())},
            "hbm": {"achieved_gbs": cycle_gbs, "peak_gbs": peak, "frac": cycle_gbs / peak,
                    "algo_bytes_per_zone_cycle": ALGO_BYTES[mode], "peak_source": peak_src}}


def golden_check(name, S):
    """Run the config's full golden length from the Sedov start (a fresh context) and
    count the fields whose SHA-256 differs from the oracle's digest (tests/golden/,
    written by scripts/oracle_digests.py from the oracle only).  None if absent."""
    import hashlib
    path = os.path.join(ROOT, "tests", "golden", f"{name}.json")
    if not os.path.exists(path):
        return None
    with open(path) as f:
        g = json.load(f)
    cfg, _ = configs.config(name)
    if g.get("params") != cfg:
        return {"skipped": "golden parameters differ from the config"}
    ctx = S.Sale(cfg)
    rc, done = ctx.step(g["requested_cycles"])
    bad = [f for f, ref in g["fields"].items()
           if hashlib.sha256(ctx.get(f).ravel().tobytes()).hexdigest() != ref["sha256"]]
    clk_ok = ctx.clock() == g["clock"]
    ctx.close()
    return {"cycles": done, "status": rc, "clock_equal": clk_ok, "fields": len(g["fields"]),
            "fields_bit_mismatched": len(bad), "mismatched": bad}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="C4", choices=["C3", "C4"])
    ap.add_argument("--impl", default="auto", choices=["auto", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-allcore", type=int, default=1, help="also time one oracle per host core (0: off)")
    ap.add_argument("--no-extras", action="store_true", help="skip the P0-state, C3 and golden-check legs")
    ap.add_argument("--halo", default="copy", choices=["copy", "peer"],
                    help="per-cycle halo exchange with N > 1: NCCL send/recv (copy) or the producing kernels "
                         "storing into the neighbours' ghost planes over NVLink (peer)")
    args = ap.parse_args()
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")
    world, rank, local = dist_env()
    if args.impl == "reference":
        run_reference(args, world, rank)
        return

    import torch
    import torch.distributed as dist

    from paper_2209_01983_b200 import build as _build
    from paper_2209_01983_b200 import sale as S

    _build.build()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("gloo")  # plumbing only: id broadcast, barrier, max
    cfg, job_cycles = configs.config(args.config, world)
    cfg["halo"] = S.HALO_PEER if args.halo == "peer" else S.HALO_COPY
    nid = None
    if world > 1:
        obj = [S.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nid = obj[0]
    ctx = S.Sale(cfg, device=local, rank=rank, nranks=world, nccl_id=nid)

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    res = time_cycles(ctx, cfg, args.steps, args.warmup, world, local, barrier, max_over_ranks, S,
                      conservation=(world == 1))
    ms, launches, prof, clocks, value = res["ms"], res["launches"], res["prof"], res["clocks"], res["value"]
    gcells = cfg["nx"] * cfg["ny"] * cfg["nz"]
    local_cells = cfg["nx"] * cfg["ny"] * (ctx.k1 - ctx.k0)
    mode = cfg["rezone"]
    roofline = roofline_of(args.config, mode, prof, ms, args.steps, local_cells)

    # ---- end to end through the public API with host buffers ------------------
    e2e = None
    if args.e2e_steps > 0:
        fields = ["UX", "UY", "UZ", "MASS", "E"] + (["X", "Y", "Z"] if mode == configs.LAGRANGE else [])
        host = {}
        for f in fields:
            shape = ctx.node_shape if f in S.NODE_FIELDS else ctx.cell_shape
            host[f] = torch.empty(shape, dtype=torch.float64, pin_memory=True)
            ctx.get(f, out=host[f])
        nbytes = sum(t.numel() * 8 for t in host.values())
        barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            for f in fields:
                ctx.set(f, host[f])          # H2D: this step's inputs, pinned host
            rc, done = ctx.step(1)
            if rc:
                raise RuntimeError(f"e2e step rc={rc}")
            for f in fields:
                ctx.get(f, out=host[f])      # D2H: this step's result (the new state)
        torch.cuda.synchronize()
        wall = max_over_ranks(time.perf_counter() - t0)
        e2e = {"value": gcells * args.e2e_steps / wall, "unit": UNIT, "h2d_bytes_per_step": nbytes,
               "d2h_bytes_per_step": nbytes, "steps": args.e2e_steps,
               "what": "per step: set_field of the full state from pinned host, sale_step(1), "
                       "get_field of the full state to pinned host"}
        # the whole BASELINE job through the same calls: the state from pinned host once,
        # the config's cycles in one sale_step, the final state back to pinned host
        barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for f in fields:
            ctx.set(f, host[f])
        rc, done = ctx.step(job_cycles)
        if rc or done != job_cycles:
            raise RuntimeError(f"e2e job rc={rc} done={done}")
        for f in fields:
            ctx.get(f, out=host[f])
        torch.cuda.synchronize()
        wall = max_over_ranks(time.perf_counter() - t0)
        e2e["job"] = {"value": gcells * job_cycles / wall, "unit": UNIT, "cycles": job_cycles,
                      "h2d_bytes": nbytes, "d2h_bytes": nbytes, "seconds": wall,
                      "what": f"the {args.config} job end to end: set_field of the full state from pinned host, "
                              f"sale_step({job_cycles}), get_field of the full state to pinned host"}

    # ---- CPU oracle baseline (rank 0, N=1 only) -------------------------------
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        s, desc = sample_cfg(args.config)
        import oracle as O
        O.build()
        v, n, dt = oracle_rate(s, args.cpu_seconds)
        cpu = {"value": v, "unit": UNIT, "cores": 1, "kind": "oracle", "cpu_model": cpu_model(),
               "sample": f"{desc}; {n} cycles in {dt:.1f} s, single thread, gcc -O2 -ffp-contract=off"}
        if args.cpu_allcore:
            agg, nproc, ncore = oracle_allcore(args.config, args.cpu_seconds / 2)
            cpu["all_cores"] = {"value": agg, "unit": UNIT, "cores": ncore, "processes": nproc,
                                "what": "one single-threaded oracle process per core on the same sample, "
                                        "concurrently; sum of their rates (replica throughput)"}

    # ---- the same workload from the seeded perturbed state P0 (every node moving: no
    # quiescent cells, so no zero-operand division shortcuts), the larger single-GPU
    # config C3, and the golden-digest check of the kernels timed (N = 1 only)
    extra = {}
    if world == 1 and not args.no_extras:
        from paper_2209_01983_b200 import inputs
        pert = inputs.perturbation(cfg, 0)
        for f in ("UX", "UY", "UZ"):
            ctx.set(f, pert[f.lower()])
        if mode == configs.LAGRANGE:
            for f, d in (("X", "dx"), ("Y", "dy"), ("Z", "dz")):
                ctx.set(f, ctx.get(f) + pert[d])
        ctx.set("E", ctx.get("E") * pert["e_factor"])
        del pert
        rp = time_cycles(ctx, cfg, args.steps, 3, world, local, barrier, max_over_ranks, S)
        extra["p0_state"] = {"value": rp["value"], "ms_per_step": rp["ms"] / args.steps,
                             "kernels_ms_per_step": {k: v[0] / args.steps for k, v in rp["prof"].items()},
                             "what": "seeded perturbed state P0 (inputs.perturbation seed 0: node jitter, "
                                     "u ~ U(-1e-3, 1e-3), e x U(0.5, 1.5)): every cell active"}
    ctx.close()
    if world == 1 and not args.no_extras:
        import torch
        torch.cuda.empty_cache()
        if args.config == "C4":
            c3, _ = configs.config("C3", 1)
            c3ctx = S.Sale(c3, device=local)
            r3 = time_cycles(c3ctx, c3, args.steps, args.warmup, world, local, barrier, max_over_ranks, S,
                             conservation=True)
            lc3 = c3["nx"] * c3["ny"] * c3["nz"]
            extra["c3"] = {"workload": workload_name("C3"), "value": r3["value"], "unit": UNIT,
                           "ms_per_step": r3["ms"] / args.steps,
                           "roofline": roofline_of("C3", c3["rezone"], r3["prof"], r3["ms"], args.steps, lc3),
                           "clocks": r3["clocks"], "gpu_launches": r3["launches"],
                           "conservation": r3.get("conservation"),
                           "kernels_ms_per_step": {k: v[0] / args.steps for k, v in r3["prof"].items()}}
            c3ctx.close()
            torch.cuda.empty_cache()
        extra["golden_check"] = golden_check(args.config, S)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": "weak" if args.config == "C4" else "strong", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic",
            "config": {"workload": workload_name(args.config), "global_cells": gcells,
                       "cells_per_gpu": local_cells, "mesh": [cfg["nx"], cfg["ny"], cfg["nz"]],
                       "parallelism": f"z-slabs x{world}" if world > 1 else "single GPU",
                       "halo": args.halo if world > 1 else "none (one slab)",
                       "step": "one SALE cycle",
                       "state": f"Sedov initial state (c.6), cycles {args.warmup + 1}..{args.warmup + args.steps}"
                                " (the shock near the origin; the bulk is quiescent -- p0_state times a "
                                "fully active state)",
                       "l2": "inputs larger than L2 (state >= 1.1 GB per GPU), no flush"},
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
            "clocks": clocks,
            "kernels_ms_per_step": {k: v[0] / args.steps for k, v in prof.items()},
            "conservation": res.get("conservation"),
        }
        line.update(extra)
        print(json.dumps(line), flush=True)
    ctx.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
