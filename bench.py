#!/usr/bin/env python
"""Bench harness: mixed-precision SLDG split step on B200 (arXiv:1603.07008).

Metric (BASELINE.json): GDoF/s per advection step and achieved HBM GB/s (% of roofline).
Default workload = BASELINE configs[4] ("C5"): 4D (x1,x2,v1,v2) dimension-split step on a
128^4 grid, k=3 per dim (81 coefficients/cell), mixed precision (c_0 fp64, rest fp32),
Landau-type initial value (eps=0.01) and per-line Vlasov CFL fields.  One step
= 4 sweeps (x1, x2, v1, v2); a sweep reads and writes every stored coefficient once.
With --gpus N (torchrun) the v2 dim is block-sharded; the v2 sweep exchanges halo layers
over NCCL (strong scaling: total grid fixed).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl sldg|reference]
                  [--config c5|c4|c3|c2] [--precision mixed|fp64] [--k K]

Prints ONE JSON line on rank 0.  --impl reference times the CPU oracle (plain C, one host
core) on a bounded sample of the same workload (sampled lines of every sweep).
"""
from __future__ import annotations

import argparse
import datetime
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import sldg_inputs  # noqa: E402

CONFIGS = {
    # name: (dims, kinds, k, lo, hi, description)
    "c5": ([128, 128, 128, 128], ["x", "x", "v", "v"], 3,
           "4D split step 128^4, k=3 (BASELINE configs[4])"),
    "c4": ([64, 64, 64, 64], ["x", "x", "v", "v"], 2, "4D split step 64^4, k=2 (BASELINE configs[3])"),
    "c3": ([4096, 4096], ["x", "v"], 4, "2D 4096^2 split step (BASELINE configs[2])"),
    "c2": ([1024, 1024], ["x", "v"], 4, "2D 1024^2 split step (BASELINE configs[1])"),
}


def domain(kinds):
    lo = [0.0 if t == "x" else -6.0 for t in kinds]
    hi = [4 * np.pi if t == "x" else 6.0 for t in kinds]
    return lo, hi


def bytes_per_cell(K: int, precision: str) -> int:
    """One stored cell: fp64 c_0 + (K-1) fp32 (mixed) or K fp64."""
    return 8 + 4 * (K - 1) if precision == "mixed" else 8 * K


def memorydown(o: int, d: int) -> float:
    """8o / (8d + 4(o-d)) (Tables III-VI 'memorydown')."""
    return 8.0 * o / (8.0 * d + 4.0 * (o - d))


def load_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms.  Started before the warm-up
    steps (nvidia-smi's start-up, NVML init included, then overlaps them, not the timed region);
    summary() keeps only the samples taken between mark(True) and mark(False) -- the timed
    region -- when there are any."""

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []
        self.t_begin = None
        self.t_end = None

    def mark(self, begin: bool):  # wall-clock marks, compared with nvidia-smi's own sample timestamps
        if begin:
            self.t_begin = datetime.datetime.now()
        else:
            self.t_end = datetime.datetime.now()

    def __enter__(self):
        q = ("timestamp,clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons, masks = [], None, set(), set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        rows = []
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                ts = datetime.datetime.strptime(parts[0], "%Y/%m/%d %H:%M:%S.%f")
            except ValueError:
                ts = None
            rows.append((ts, parts[1:]))
        if self.t_begin is not None:
            t1 = self.t_end or datetime.datetime.max
            inside = [r for r in rows if r[0] is not None and self.t_begin <= r[0] <= t1]
            if inside:
                rows = inside
        for _, parts in rows:
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            masks.add(parts[2])
            for nm, v in zip(names, parts[3:7]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_min_mhz": min(sm), "sm_max_mhz": mx,
                "reasons": sorted(reasons), "active_masks": sorted(masks), "samples": len(sm)}


# ---------------------------------------------------------------------------------------------
# CPU oracle (cpu_baseline leg and --impl reference): sampled lines of every sweep
# ---------------------------------------------------------------------------------------------
def oracle_line_specs(dims, kinds, k, lines_per_sweep: int, seed: int = 1603, eps: float = 0.01):
    """Random lines of every sweep of the split step: (sweep, dim, perpendicular cell base,
    CFL number, input slot).  At most 64 distinct input lines per sweep are generated (the
    oracle's time does not depend on the values); line i uses input slot i % 64."""
    D = len(dims)
    lo, hi = domain(kinds)
    rng = np.random.default_rng(seed)
    S = np.cumprod([1] + list(dims[:-1]))
    specs = []
    for si, (d, field, mask) in enumerate(sldg_inputs.vlasov_fields(dims, kinds, lo, hi, eps=eps)):
        fd = [e for e in range(D) if mask >> e & 1]
        bases = {}
        for i in range(lines_per_sweep):
            perp = {e: int(rng.integers(0, dims[e])) for e in range(D) if e != d}
            fi, st = 0, 1
            for e in fd:
                fi += perp[e] * st
                st *= dims[e]
            slot = i % 64
            if slot not in bases:
                bases[slot] = int(sum(perp[e] * S[e] for e in perp))
            specs.append((si, d, bases[slot], float(field[fi]), slot))
    return specs


def oracle_run_specs(dims, k, precision, specs, seed: int = 1603):
    """Run oracle.advect on each spec'd line (inputs: the parity generator's values of that
    line).  Returns (timed seconds of the oracle calls only, DoF, per-line output digests)."""
    import hashlib

    import oracle  # test infrastructure; only the cpu_baseline / reference legs of bench.py use it

    D, K = len(dims), k ** len(dims)
    nd = 1 if precision == "mixed" else K
    S = np.cumprod([1] + list(dims[:-1]))
    cache = {}
    secs, dofs, digests = 0.0, 0, []
    for si, d, base, nu, slot in specs:
        key = (si, slot)
        if key not in cache:
            cells = base + np.arange(dims[d]) * S[d]
            cache[key] = oracle.round_layout(sldg_inputs.random_coeffs(dims, k, seed, cells=cells), K, nd)
        ldims = [1] * D
        ldims[d] = dims[d]
        t0 = time.perf_counter()
        out = oracle.advect(cache[key], ldims, k, d, shift=nu, n_double=nd)
        secs += time.perf_counter() - t0
        dofs += dims[d] * K
        digests.append(hashlib.blake2b(out.tobytes(), digest_size=8).digest())
    return secs, dofs, digests


def _oracle_worker(a):
    dims, k, precision, specs = a
    return oracle_run_specs(dims, k, precision, specs)


def host_cpu():
    """nproc (the cores this process may use) and the CPU model (lscpu)."""
    cores = len(os.sched_getaffinity(0))
    model = None
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for ln in out.splitlines():
            if ln.startswith("Model name:"):
                model = ln.split(":", 1)[1].strip()
    except Exception:
        pass
    if model is None:
        try:
            with open("/proc/cpuinfo") as f:
                model = next(ln.split(":", 1)[1].strip() for ln in f if ln.startswith("model name"))
        except Exception:
            model = "unknown"
    return cores, model


def oracle_baseline(dims, kinds, k, precision, lines_per_sweep: int, eps: float = 0.01):
    """SURVEY 8(d) 'Timing the oracle': the same bounded sample of lines timed on 1 host core and
    on all host cores (a process pool over independent lines; each line's result is
    bit-identical to the 1-core leg's, checked by digest).  Throughput = DoF / oracle seconds
    (1 core) and DoF / max over workers of their oracle seconds (all cores, concurrent)."""
    import multiprocessing as mp
    from concurrent.futures import ProcessPoolExecutor

    specs = oracle_line_specs(dims, kinds, k, lines_per_sweep, eps=eps)
    secs1, dofs, dig1 = oracle_run_specs(dims, k, precision, specs)
    cores, model = host_cpu()
    chunks = [specs[i::cores] for i in range(cores)]  # interleaved: every worker sees every sweep
    with ProcessPoolExecutor(max_workers=cores, mp_context=mp.get_context("spawn")) as ex:
        list(ex.map(_oracle_worker, [(dims, k, precision, c[:8]) for c in chunks]))  # start + warm workers
        t0 = time.perf_counter()
        res = list(ex.map(_oracle_worker, [(dims, k, precision, c) for c in chunks]))
        wall = time.perf_counter() - t0
    digp = [None] * len(specs)
    for i, (_, _, dg) in enumerate(res):
        digp[i::cores] = dg
    secs_all = max(r[0] for r in res)
    return {"value": dofs / secs1 / 1e9, "unit": "GDoF/s", "cores": 1, "kind": "oracle",
            "value_all_cores": dofs / secs_all / 1e9, "cores_all": cores,
            "value_all_cores_wall": dofs / wall / 1e9,
            "bit_identical_all_vs_1": digp == dig1, "cpu_model": model, "nproc": cores,
            "sample": f"{lines_per_sweep} random lines per sweep x {len(dims)} sweeps of the same workload "
                      f"({dofs} DoF; 1 core {secs1:.1f} s, {cores} cores {secs_all:.2f} s of oracle time per "
                      f"worker, {wall:.2f} s wall incl. input generation); plain C oracle, -O2 -ffp-contract=off"}


def run_reference(args, dims, kinds, k, cfg_json):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    lines = args.ref_lines
    for w in range(args.warmup):
        oracle_run_specs(dims, k, args.precision, oracle_line_specs(dims, kinds, k, max(1, lines // 8), seed=99 + w))
    t_total, dof_total = 0.0, 0
    for s in range(args.steps):
        t, n, _ = oracle_run_specs(dims, k, args.precision, oracle_line_specs(dims, kinds, k, lines, seed=1603 + s))
        t_total += t
        dof_total += n
    value = dof_total / t_total / 1e9
    bpd = bytes_per_cell(k ** len(dims), args.precision) / k ** len(dims)
    sample = (f"{lines} random lines per sweep x {len(dims)} sweeps per step of the {args.config} workload "
              f"(oracle.advect on each line, same k, same per-line CFL); timed oracle calls only")
    out = {
        "impl": "reference", "metric": "GDoF/s per advection sweep (split step of all dims)",
        "value": value, "unit": "GDoF/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": t_total / args.steps * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": cfg_json,
        "hbm_gbs_equiv": value * bpd * 2,
        "cpu_baseline": {"value": value, "unit": "GDoF/s", "cores": 1, "kind": "oracle", "sample": sample,
                         "cpu_model": host_cpu()[1], "nproc": host_cpu()[0]},
        "e2e": {"value": value, "unit": "GDoF/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(out))
    return 0


# ---------------------------------------------------------------------------------------------
def self_launch(n: int) -> int:
    """`python bench.py --gpus N` without a launcher: start N ranks (one process per GPU) with
    torch.distributed.run on 127.0.0.1, exactly as the driver's torchrun command does."""
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="sldg", choices=["sldg", "reference"])
    ap.add_argument("--config", default="c5", choices=sorted(CONFIGS))
    ap.add_argument("--precision", default="mixed", choices=["mixed", "fp64"])
    ap.add_argument("--k", type=int, default=None)
    ap.add_argument("--eps", type=float, default=0.01)
    ap.add_argument("--ref-lines", type=int, default=4096)
    ap.add_argument("--cpu-lines", type=int, default=45000)  # ~15 s of oracle time on the GPU box
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--compare-fp64", action=argparse.BooleanOptionalAction, default=True,
                    help="also time the all-fp64 layout on a slab of the workload (mixed_vs_fp64)")
    ap.add_argument("--vlasov", action=argparse.BooleanOptionalAction, default=True,
                    help="also time the Vlasov-Poisson Strang step (NEXT-2) on the same grid")
    ap.add_argument("--kernel-events", action=argparse.BooleanOptionalAction, default=True,
                    help="diagnostic: --no-kernel-events times the step without the per-launch CUDA events "
                         "(no roofline.achieved)")
    ap.add_argument("--graph", action=argparse.BooleanOptionalAction, default=True,
                    help="replay the timed steps from a CUDA graph of one split step (1 GPU)")
    ap.add_argument("--sweeps", default=None, help="comma list of dims to run (default: all)")
    ap.add_argument("--dims", default=None, help="override grid extents (profiling slabs), e.g. 128,128,128,16")
    ap.add_argument("--force-halo", action="store_true",
                    help="diagnostic: run the layer-dim sweep through the sharded halo path on one GPU")
    ap.add_argument("--nccl-self", action="store_true",
                    help="diagnostic (with --force-halo): the self halo through NCCL send/recv")
    ap.add_argument("--peer-halo", action="store_true",
                    help="pad layers mapped onto the ring neighbours' edge layers (SLDG_DIST_PEER_HALO); with one "
                         "GPU implies --force-halo (the rank's own edges)")
    ap.add_argument("--fuse-x", action=argparse.BooleanOptionalAction, default=True,
                    help="run the dim-0 and dim-1 sweeps as one fused pass (sldg_advect_pair_device, NEXT-4)")
    ap.add_argument("--timeline", action="store_true",
                    help="record the device timeline of one step (sweeps + halo exchanges) into the JSON")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return self_launch(args.gpus)
    if "WORLD_SIZE" in os.environ and int(os.environ["WORLD_SIZE"]) != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={os.environ['WORLD_SIZE']}")

    dims, kinds, k0, desc = CONFIGS[args.config]
    if args.dims:
        dims = [int(x) for x in args.dims.split(",")]
        assert len(dims) == len(kinds)
        desc = f"{desc} -- PROFILING SLAB dims={dims}"
    k = args.k or k0
    D, K = len(dims), k ** len(dims)
    cells = int(np.prod(dims))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if args.peer_halo and world == 1:
        args.force_halo = True
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    sweep_dims = list(range(D)) if args.sweeps is None else [int(x) for x in args.sweeps.split(",")]
    cfg_json = {"workload": f"{args.config}: {desc}", "dims": dims, "k": k, "coeffs_per_cell": K,
                "precision": args.precision,
                "storage": "c0 fp64 + other coefficients fp32" if args.precision == "mixed" else "all fp64",
                "ic": f"landau eps={args.eps}", "sweeps_per_step": len(sweep_dims),
                "parallelism": f"shard v{D // 2 if D > 2 else 1} (dim {D - 1}) x{world}" if world > 1 else "1 GPU",
                "l2": "inputs larger than L2 (no flush needed)" if cells * bytes_per_cell(K, args.precision) > 4 * 126e6
                else "source + destination arrays exceed L2 (126 MB) but one array is comparable: partial "
                     "L2 residency between sweeps",
                "dt": 0.1}
    if args.impl == "reference":
        return run_reference(args, dims, kinds, k, cfg_json)

    import torch
    import torch.distributed as dist

    from paper_1603_07008_b200 import Grid, sldg

    torch.cuda.set_device(local_rank)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        uid = [sldg.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        uid = uid[0]
    else:
        uid = None

    lo, hi = domain(kinds)
    g = Grid(dims, k, lo=lo, hi=hi, precision=args.precision, rank=rank, world=world, unique_id=uid,
             max_halo=2, force_halo=args.force_halo, nccl_self=args.nccl_self, peer_halo=args.peer_halo)
    terms = sldg_inputs.landau_terms(dims, k, kinds, lo, hi, eps=args.eps)
    g.fill_separable(terms)
    sweeps = [s for s in sldg_inputs.vlasov_fields(dims, kinds, lo, hi, eps=args.eps) if s[0] in sweep_dims]
    dev_fields = [torch.tensor(f, dtype=torch.float64, device="cuda") for _, f, _ in sweeps]
    bounds = [(float(np.min(f)), float(np.max(f))) for _, f, _ in sweeps]
    stream = torch.cuda.ExternalStream(g.stream())
    torch.cuda.synchronize()
    sharded = world > 1 or args.force_halo

    fuse = args.fuse_x and len(sweeps) >= 2 and sweeps[0][0] == 0 and sweeps[1][0] == 1

    def step():
        first = 0
        if fuse:  # x1 + x2 in one pass over HBM (sldg_advect_pair_device)
            g.advect_pair_device(dev_fields[0].data_ptr(), sweeps[0][2], dev_fields[1].data_ptr(), sweeps[1][2])
            first = 2
        for (d, _, m), tf, (b0, b1) in list(zip(sweeps, dev_fields, bounds))[first:]:
            if sharded:  # the field's bound sizes the halo on the host: no device -> host read
                g.advect_device_bounded(d, tf.data_ptr(), m, b0, b1)
            else:
                g.advect_device(d, tf.data_ptr(), m)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        g.sync()

    clk = ClockSampler(local_rank).__enter__()  # nvidia-smi starts during the warm-up
    mass0 = g.mass()
    for _ in range(args.warmup):
        step()
    barrier()
    # per-sweep kernel durations (CUDA events the library records around each sweep launch on
    # its stream), from one eager step outside the timed region when the timed steps replay a
    # graph, else from the timed steps themselves
    # graphs only where the host's per-call cost shows (steps of < 1e9 DoF: C2-C4); C5's timed
    # region stays eager so the per-kernel events are taken inside it
    # (one GPU only: sharded grids capture too -- tested with the NCCL self-exchange -- but real
    # multi-rank NCCL inside a capture has not run on hardware here)
    use_graph = args.graph and world == 1 and len(sweeps) % 2 == 0 and len(sweeps) * cells * K < 1e9
    graph = None
    if use_graph:
        g.kernel_time(reset=True)
        g.profile(True)
        for _ in range(2):
            step()
        barrier()
        g.profile(False)
        kt_all = g.kernel_time(-1)
        per_dim = {d: g.kernel_time(d) for d in sweep_dims}
        if fuse:
            per_dim = {d: v for d, v in per_dim.items() if v[1] > 0}
            per_dim[-2] = g.kernel_time(-2)
        g_kernel_names = {d: (g.sweep_kernel(d) if d >= 0 else "sweep_fused01_kernel") for d in per_dim}
        g.graph_begin()
        step()
        graph = g.graph_end()
        graph.launch()  # warm the graph once
        barrier()
    # ---------------------------------------------------------------- device-timed region
    if not use_graph:
        g.kernel_time(reset=True)
        g.profile(args.kernel_events)
    launches0 = g.launch_count()
    # one event between consecutive steps (same stream, no host sync): per-step times for the
    # median of the K repetitions (SURVEY 8(d) "median of >= 5 repetitions")
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    e0, e1 = evs[0], evs[-1]
    barrier()
    clk.mark(True)
    with torch.cuda.stream(stream):
        e0.record(stream)
    for i in range(args.steps):
        if graph is not None:
            graph.launch()
        else:
            step()
        with torch.cuda.stream(stream):
            evs[i + 1].record(stream)
    barrier()
    clk.mark(False)
    clk.__exit__(None, None, None)
    ms = e0.elapsed_time(e1)
    step_times = torch.tensor([evs[i].elapsed_time(evs[i + 1]) for i in range(args.steps)], dtype=torch.float64,
                              device="cuda")
    launches = g.launch_count() - launches0
    if not use_graph:
        g.profile(False)
        kt_all = g.kernel_time(-1)
        per_dim = {d: g.kernel_time(d) for d in sweep_dims}
        if fuse:
            per_dim = {d: v for d, v in per_dim.items() if v[1] > 0}
            per_dim[-2] = g.kernel_time(-2)
        g_kernel_names = {d: (g.sweep_kernel(d) if d >= 0 else "sweep_fused01_kernel") for d in per_dim}
    if graph is not None:
        graph.destroy()
    t = torch.tensor([ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.all_reduce(step_times, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    step_times = step_times.cpu().tolist()
    mass1 = g.mass()
    timeline = None
    if args.timeline:  # one eager step with every sweep launch and halo exchange on the device clock
        g.profile(True)
        g.timeline(reset=True)
        step()
        timeline = [{"kind": "halo" if kd == -1 else "fused dims 0+1" if kd == -2 else f"sweep dim {kd}", "t0_ms": a, "t1_ms": b}
                    for kd, a, b in g.timeline(reset=True)]
        g.profile(False)
        g.kernel_time(reset=True)

    # ---------------------------------------------------------------- end-to-end (C ABI, host buffers)
    e2e = None
    if not args.no_e2e:
        pinned = []
        for _, f, _ in sweeps:
            pt = torch.empty(len(f), dtype=torch.float64, pin_memory=True)
            pt.numpy()[:] = f
            pinned.append(pt)
        h2d = sum(p.numel() * 8 for p in pinned)
        eclk = ClockSampler(local_rank).__enter__()
        barrier()
        eclk.mark(True)
        t0 = time.perf_counter()
        for _ in range(args.steps):
            first = 0
            if fuse:
                g.advect_pair(0.0, pinned[0].numpy(), sweeps[0][2], 0.0, pinned[1].numpy(), sweeps[1][2])
                first = 2
            for (d, _, m), p in list(zip(sweeps, pinned))[first:]:
                g.advect(d, field=p.numpy(), field_mask=m)
            g.mass()  # D2H read of the step's diagnostic (blocking)
        barrier()
        e2e_s = time.perf_counter() - t0
        eclk.mark(False)
        eclk.__exit__(None, None, None)
        te = torch.tensor([e2e_s], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e2e_s = float(te.item())
        e2e = {"value": len(sweeps) * cells * K * args.steps / e2e_s / 1e9, "unit": "GDoF/s",
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": 8 * world,
               "api": "sldg_advect (host pinned CFL fields, one per sweep) + sldg_mass (D2H) per step",
               "clocks": eclk.summary()}

    launch_steps = 2 if use_graph else args.steps  # steps the per-kernel events cover
    if rank == 0:
        peak, peak_src = load_peak()
        step_ms = ms_max / args.steps
        dofs_per_step = len(sweeps) * cells * K
        alg_bytes_step = len(sweeps) * 2 * cells * bytes_per_cell(K, args.precision)
        value = dofs_per_step / (step_ms * 1e-3) / 1e9
        # per kernel function (a template instance may serve several sweep dims): launches, time,
        # algorithmic bytes; the dominant kernel is the one with the largest total time (rank 0)
        kname = {d: (g_kernel_names[d]) for d in per_dim}
        kernels = {}
        for d, (ms_d, n_d, b_d) in per_dim.items():
            e = kernels.setdefault(kname[d], {"ms": 0.0, "launches": 0, "bytes": 0.0, "dims": []})
            e["ms"] += ms_d
            e["launches"] += n_d
            e["bytes"] += b_d
            e["dims"].append(d if d >= 0 else "0+1")
        dom_name = max(kernels, key=lambda kn: kernels[kn]["ms"])
        dk = kernels[dom_name]
        d_ms, d_n, d_bytes = dk["ms"], dk["launches"], dk["bytes"]
        achieved = (d_bytes / d_n) / (d_ms / d_n * 1e-3) / 1e9 if d_n else None
        dom = max((d for d in per_dim if kname[d] == dom_name), key=lambda d: per_dim[d][0])
        traffic, traffic_all = None, None
        try:
            with open(os.path.join(ROOT, "profiles", "ncu_dram.json")) as f:
                nd = json.load(f)
            key = f"{args.config}_{args.precision}_k{k}_dim{dom}" if dom >= 0 else f"{args.config}_{args.precision}_k{k}_fused01"
            traffic = nd.get(key)
            traffic_all = {str(d): nd.get(f"{args.config}_{args.precision}_k{k}_dim{d}") for d in sweep_dims}
        except Exception:
            traffic_all = None
        # secondary roofline: fp64-pipe and XU (F2F) activity of the dominant kernel
        # from the ncu launch list of this config (profiles/ncu_pipe.json)
        secondary = {"bound": "fp64 pipe", "dfma_per_cell_per_sweep": 2 * k * K,
                     "fp64_pipe_pct": None, "xu_pct": None,
                     "source": "profiles/ncu_pipe.json: sm__pipe_fp64_cycles_active / sm__inst_executed_pipe_xu "
                               "(% of peak sustained active) of the launch-list pass of this config"}
        try:
            with open(os.path.join(ROOT, "profiles", "ncu_pipe.json")) as f:
                npj = json.load(f)
            key = f"{args.config}_{args.precision}_k{k}_dim{dom}" if dom >= 0 else f"{args.config}_{args.precision}_k{k}_fused01"
            if key in npj:
                secondary["fp64_pipe_pct"] = npj[key]["fp64_pipe_pct"]
                secondary["xu_pct"] = npj[key]["xu_pct"]
        except Exception:
            pass
        cpu = None
        if not args.no_cpu_baseline and world == 1:
            cpu = oracle_baseline(dims, kinds, k, args.precision, args.cpu_lines, eps=args.eps)
        out = {
            "metric": "GDoF/s per advection sweep (split step of all dims)",
            "value": value, "unit": "GDoF/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": step_ms, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f64",  # arithmetic type; storage is config.storage
            "data": "synthetic (Landau-type IC, Vlasov CFL fields)", "config": cfg_json,
            "hbm_gbs": alg_bytes_step / (step_ms * 1e-3) / 1e9 / world,
            "hbm_frac_of_peak": alg_bytes_step / (step_ms * 1e-3) / 1e9 / world / peak,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": (achieved / peak) if achieved else None, "traffic": traffic,
                         "traffic_per_sweep": traffic_all,
                         "traffic_source": "profiles/ncu_dram.json: dram__bytes_read.sum + dram__bytes_write.sum "
                                           "per launch of each sweep dim, ncu launch list of this config",
                         "algorithmic_bytes_per_sweep": 2 * cells * bytes_per_cell(K, args.precision),
                         "kernel": f"{dom_name} (sweeps along dims {dk['dims']})",
                         "share_of_kernel_time": d_ms / max(1e-12, sum(e["ms"] for e in kernels.values())),
                         "peak_source": peak_src,
                         "frac_of_spec_8000": (achieved / 8000.0) if achieved else None,
                         "bytes_per_launch": d_bytes / d_n if d_n else None,
                         "launch_timing": ("CUDA events around each sweep launch in 2 eager steps before the "
                                           "graph-replayed timed region") if use_graph else
                                          "CUDA events around each sweep launch inside the timed region",
                         "avg_launch_ms": d_ms / d_n if d_n else None,
                         "secondary": secondary,
                         "kernels": {kn: {"dims": e["dims"], "launches_per_step": e["launches"] / max(1, launch_steps),
                                          "ms_per_launch": e["ms"] / max(1, e["launches"]),
                                          "achieved_gbs": e["bytes"] / (e["ms"] * 1e-3) / 1e9 if e["ms"] else None,
                                          "frac": (e["bytes"] / (e["ms"] * 1e-3) / 1e9 / peak) if e["ms"] else None,
                                          "share": e["ms"] / max(1e-12, sum(x["ms"] for x in kernels.values()))}
                                     for kn, e in kernels.items()},
                         "bytes_note": ("algorithmic bytes = one read + one write of every stored coefficient per "
                                        "launch (SURVEY 8(d)); the fused x1+x2 launch does two sweeps with ONE read + "
                                        "write, so its per-sweep-equivalent rate is twice its achieved GB/s") if fuse else
                                       "algorithmic bytes = one read + one write of every stored coefficient per sweep"},
            "fused_x": fuse,
            "sweeps": {(str(d) if d >= 0 else "fused01"): {"ms_per_launch": per_dim[d][0] / max(1, per_dim[d][1]),
                                "gbs": (per_dim[d][2] / (per_dim[d][0] * 1e-3) / 1e9) if per_dim[d][0] else None}
                       for d in per_dim},
            "kernel_share_of_step": (kt_all[0] / max(1, kt_all[1]) * len(sweeps) * args.steps) / ms if ms else None,
            "timed_steps": "CUDA graph of one split step, replayed" if use_graph else "eager calls",
            "step_ms_median": statistics.median(step_times), "step_ms_min": min(step_times),
            "step_ms_max": max(step_times),
            "gdofs_median_step": dofs_per_step / (statistics.median(step_times) * 1e-3) / 1e9,
            "gpu_launches": launches,
            "mass_rel_drift": abs(mass1 - mass0) / abs(mass0),
            "clocks": clk.summary(),
            "e2e": e2e,
            "cpu_baseline": cpu,
        }
        if timeline is not None:
            out["timeline"] = timeline
        if args.force_halo:
            out["config"]["diagnostic"] = "forced halo path on one GPU" + (" (NCCL self)" if args.nccl_self else "") \
                + (" (peer-mapped pads)" if args.peer_halo else "")
        if args.peer_halo:
            out["config"]["halo"] = "peer-mapped"
    vp_res = None
    if args.vlasov and world == 1 and args.sweeps is None:
        vp_res = time_vlasov(g, stream, dims, kinds, k)
    g.destroy()
    del dev_fields
    if rank == 0:
        if vp_res is not None:
            out["vlasov_poisson_step"] = vp_res
        if args.compare_fp64 and world == 1:
            out["mixed_vs_fp64"] = compare_precisions(args, dims, kinds, k)
        print(json.dumps(out))
    if world > 1:
        dist.destroy_process_group()
    return 0


def time_vlasov(g, stream, dims, kinds, k, steps=3, dt=0.1):
    """NEXT-2: the Vlasov-Poisson Strang step (x sweeps dt/2, density, field, v sweeps dt,
    x sweeps dt/2; sldg_vp_step) on the benchmark grid, and the density + field solve alone.
    Device time (CUDA events on the grid stream)."""
    import torch

    from paper_1603_07008_b200 import VlasovPoisson

    dx = kinds.count("x")
    vp = VlasovPoisson(g, dx)
    vp.step(dt)  # warm-up (also builds the tensor maps of every sweep)
    vp.field_async()
    g.sync()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    with torch.cuda.stream(stream):
        ev[0].record(stream)
    for _ in range(steps):
        vp.step(dt)
    with torch.cuda.stream(stream):
        ev[1].record(stream)
    for _ in range(steps):
        vp.field_async()
    with torch.cuda.stream(stream):
        ev[2].record(stream)
    g.sync()
    step_ms = ev[0].elapsed_time(ev[1]) / steps
    field_ms = ev[1].elapsed_time(ev[2]) / steps
    cells, K = int(np.prod(dims)), k ** len(dims)
    w = vp.step(dt, energy=True)
    # NEXT-3: the same step with Gauss-node x sweeps, and one nodal x1 sweep alone
    vp.set_nodal(True)
    vp.step(dt)
    g.sync()
    with torch.cuda.stream(stream):
        ev[0].record(stream)
    for _ in range(steps):
        vp.step(dt)
    with torch.cuda.stream(stream):
        ev[1].record(stream)
    g.sync()
    nodal_ms = ev[0].elapsed_time(ev[1]) / steps
    g.profile(True)
    g.kernel_time(reset=True)
    nv = dims[dx]
    xg = np.polynomial.legendre.leggauss(k)[0]
    lo_v, hi_v = -6.0, 6.0
    hv = (hi_v - lo_v) / nv
    vc = lo_v + (np.arange(nv) + 0.5) * hv
    nodal_nu = ((vc[:, None] + xg[None, :] * hv / 2) * dt / (4 * np.pi / dims[0])).reshape(-1)
    d_nodal = torch.tensor(nodal_nu, dtype=torch.float64, device="cuda")
    for _ in range(steps):
        g.advect_vnodes_device(0, dx, d_nodal.data_ptr())
    g.sync()
    v_ms, v_n, v_bytes = g.kernel_time(0)
    g.profile(False)
    vp.destroy()
    nodal = {"ms_per_step": nodal_ms, "x_sweep_kernel_ms": v_ms / max(1, v_n),
             "x_sweep_gbs": (v_bytes / (v_ms * 1e-3) / 1e9) if v_ms else None,
             "x_sweep_kernel": "vnode_sweep_multi (Gauss-node x1 sweep, V7; 2 cells per thread)"}
    return {"ms_per_step": step_ms, "nodal_x": nodal, "sweeps_per_step": 3 * dx, "density_and_field_ms": field_ms,
            "field_share_of_step": field_ms / step_ms,
            "gdofs_per_sweep": 3 * dx * cells * K / (step_ms * 1e-3) / 1e9,
            "electric_energy": w, "dt": dt,
            "field_solver": "1D: exact DG antiderivative (V3)" if dx == 1 else "2D: spectral on cell means (V4)"}


def compare_precisions(args, dims, kinds, k):
    """North_star 'mixed >= 1.6x faster than all-fp64': the same split step on both storage
    layouts, on a slab of the workload small enough that the fp64 pair fits one GPU (the outer
    dim cut to 32 layers).  Device time over the same sweeps, CUDA events on the grid stream."""
    import torch

    from paper_1603_07008_b200 import Grid

    sdims = list(dims)
    if int(np.prod(sdims)) * 8 * k ** len(dims) * 2 > 120e9:
        sdims[-1] = 32
    lo, hi = domain(kinds)
    res = {"slab_dims": sdims, "fused_x": bool(args.fuse_x)}
    for prec in ["mixed", "fp64"]:
        g = Grid(sdims, k, lo=lo, hi=hi, precision=prec)
        g.fill_separable(sldg_inputs.landau_terms(sdims, k, kinds, lo, hi, eps=args.eps))
        sweeps = sldg_inputs.vlasov_fields(sdims, kinds, lo, hi, eps=args.eps)
        dfs = [torch.tensor(f, dtype=torch.float64, device="cuda") for _, f, _ in sweeps]
        torch.cuda.synchronize()
        stream = torch.cuda.ExternalStream(g.stream())
        fuse = args.fuse_x and len(sweeps) >= 2 and sweeps[0][0] == 0 and sweeps[1][0] == 1

        def step():  # the same split step as the timed one (fused x pair when enabled)
            first = 0
            if fuse:
                g.advect_pair_device(dfs[0].data_ptr(), sweeps[0][2], dfs[1].data_ptr(), sweeps[1][2])
                first = 2
            for (d, _, m), tf in list(zip(sweeps, dfs))[first:]:
                g.advect_device(d, tf.data_ptr(), m)

        for _ in range(2):
            step()
        g.sync()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            e0.record(stream)
        for _ in range(3):
            step()
        with torch.cuda.stream(stream):
            e1.record(stream)
        g.sync()
        res[f"{prec}_ms_per_step"] = e0.elapsed_time(e1) / 3
        g.destroy()
        del dfs
        torch.cuda.synchronize()
    res["speedup"] = res["fp64_ms_per_step"] / res["mixed_ms_per_step"]
    K = k ** len(dims)
    res["memorydown"] = bytes_per_cell(K, "fp64") / bytes_per_cell(K, "mixed")
    return res


if __name__ == "__main__":
    sys.exit(main())
