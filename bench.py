"""Benchmark: decompose + recompose throughput (GB/s of input) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

`--gpus N` (N > 1) outside torchrun relaunches itself under
torch.distributed.run with N ranks on 127.0.0.1.

One step = decompose + recompose of one 513^3 fp32 field (BASELINE.json
config 2 shape/distribution; config 5a's per-field unit when N > 1) with the
input resident in HBM.  Under torchrun every rank processes its own field
(per-rank seed) — batch sharding with no collective on the data path, so
`scaling` is "weak" and `value` = all ranks' input bytes / max-over-ranks
time.  Rank 0 prints one JSON line.

`--impl reference` times the reference's own CPU implementation
(oracle/_ref/libmgrx_ref.so, the unmodified reference compiled from its
sources; falls back to the pinned oracle port if that library is absent) on
the host cores, rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

DIMS = (513, 513, 513)
FIELD_DTYPE = "f32"
WORKLOAD = "config2: 513^3 fp32 field (16 bumps + 8 oblique sine modes + 1e-4 noise), full decompose + recompose (stop 0)"
METRIC = "decompose+recompose GB/s of input per GPU and % of HBM roofline; 1/2/4/8 GPU"


def hierarchy_bytes(dims, esize):
    """Algorithmic bytes per direction: sum_{l=1..L} 2 * s * #N_l."""
    import numpy as np

    from paper_2010_05872_b200 import GridHierarchy

    h = GridHierarchy.create(dims)
    return sum(2 * esize * h.node_count(l) for l in range(1, h.num_levels() + 1)), h


def measured_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        rows = [r for r in self.rows if len(r) == 6]
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[2 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


def dist_init(backend="nccl"):
    """One process per GPU (torchrun env).  Batch sharding: rank r runs its
    own field (seed r); the only collectives are the timing barrier and the
    max-over-ranks of the device time.  `backend` gloo is for the CPU tests."""
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if ws > 1:
        import torch.distributed as dist

        dist.init_process_group(backend=backend)
        # one line per rank on stderr: the rank count the driver can check
        print(f"[bench] rank {rank}/{ws} local_rank {local} backend {dist.get_backend()} "
              f"master {os.environ.get('MASTER_ADDR')}:{os.environ.get('MASTER_PORT')}", file=sys.stderr, flush=True)
    return ws, rank, local


def self_launch(nproc, argv):
    """`python bench.py --gpus N` outside torchrun: relaunch this script
    under torch.distributed.run with N ranks (one per GPU) on 127.0.0.1 and
    return its exit code (rank 0's JSON line goes to stdout)."""
    import socket

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + list(argv)
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "WARN")
    env.setdefault("OMP_NUM_THREADS", "1")
    print("[bench] launching " + " ".join(cmd), file=sys.stderr, flush=True)
    return subprocess.call(cmd, env=env)


def dist_selftest(args):
    """CPU check of the N > 1 plumbing (gloo): every rank reports a fixed
    per-rank time, rank 0 prints the JSON line exactly as run_ours would
    aggregate it (used by tests/test_dist_host.py)."""
    ws, rank, local = dist_init(backend="gloo")
    ms = 1.0 + rank
    barrier(ws)
    m = max_over_ranks(ms, ws, device="cpu")
    if rank == 0:
        print(json.dumps({"metric": METRIC, "value": aggregate_gbs(ws, 1e9, m), "unit": "GB/s", "n_gpus": ws,
                          "ms_per_step": m, "selftest": True}), flush=True)
    if ws > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


def field_seed(rank):
    """Seed of the field a rank processes (config 5a: seed = field index)."""
    return rank


def max_over_ranks(x, ws, device="cuda"):
    if ws == 1:
        return x
    import torch
    import torch.distributed as dist

    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def aggregate_gbs(ws, nbytes_per_rank, ms_max):
    """Whole-job throughput: bytes of all ranks over the slowest rank's time."""
    return ws * nbytes_per_rank / (ms_max * 1e-3) / 1e9


def barrier(ws):
    if ws > 1:
        import torch.distributed as dist

        dist.barrier()


# --------------------------------------------------------------- reference

def run_reference(args, ws, rank):
    """The reference's own CPU path on all host threads: each thread runs
    mgrx::decompose + mgrx::recompose (transform.hpp:509,517) on its own
    513^3 fp32 field, one field per thread per step."""
    if rank != 0:
        return
    import ctypes
    import numpy as np

    from oracle.oracle import Oracle, Reference, reference_available

    lib = Reference() if reference_available() else Oracle()
    kind = "reference" if reference_available() else "port"
    ncpu = physical_cores()
    try:
        import psutil

        avail = psutil.virtual_memory().available
    except Exception:
        avail = 16 << 30
    per_field = 4 * 540_000_000  # input + output + reference field copy + fp64 correction scratch
    threads = max(1, min(ncpu, int(avail * 0.6 // per_field), args.ref_threads or ncpu))
    import torch

    from synthetic_fields import config2_field

    fields = [config2_field(DIMS, seed=i).numpy() for i in range(threads)]
    outs = [np.empty(f.size, dtype=np.float32) for f in fields]

    def work(i):
        c = lib.decompose(fields[i])
        outs[i] = lib.recompose(c, DIMS)

    def step():
        ts = [threading.Thread(target=work, args=(i,)) for i in range(threads)]
        for t in ts:
            t.start()
        for t in ts:
            t.join()

    for _ in range(args.warmup_ref):
        step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    dt = time.perf_counter() - t0
    nbytes = threads * fields[0].nbytes * args.steps
    value = nbytes / dt / 1e9
    err = float(np.max(np.abs(outs[0].reshape(DIMS) - fields[0])))
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": dt / args.steps * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": WORKLOAD, "field": list(DIMS), "field_dtype": FIELD_DTYPE,
                   "parallelism": f"{threads} host threads, one field each"},
        "cpu_baseline": {"value": value, "unit": "GB/s", "cores": threads, "kind": kind,
                         "sample": f"{threads} x 513^3 f32 decompose+recompose per step, "
                                   f"{args.warmup_ref} untimed warm-up steps",
                         "cpu": _cpu_model(), "logical_cpus": os.cpu_count()},
        "e2e": {"value": value, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "roundtrip_linf": err,
    }
    print(json.dumps(line), flush=True)


def physical_cores():
    """Physical core count of the host (P = physical cores,
    not logical CPUs)."""
    try:
        import psutil

        n = psutil.cpu_count(logical=False)
        if n:
            return int(n)
    except Exception:
        pass
    try:
        cores = set()
        phys = None
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("physical id"):
                    phys = line.split(":", 1)[1].strip()
                elif line.startswith("core id"):
                    cores.add((phys, line.split(":", 1)[1].strip()))
        if cores:
            return len(cores)
    except Exception:
        pass
    return os.cpu_count() or 1


def _cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def cpu_baseline_sample(field_np, mg=None, wsp=None, field=None, h=None):
    """Reference CPU decompose+recompose of the same field on 1 core (the
    library is single-threaded by contract).  With the GPU
    objects given, the reference's coefficients also serve as the parity
    check of the bench field (north_star's bars): coefficient error over the
    range, and for tau in {1e-2, 1e-3, 1e-4} * range the label flips against
    the reference's quantize (each within 1 ulp of a bin edge) and the
    L_inf / tau of the GPU dequantize + recompose."""
    import numpy as np

    from oracle.oracle import Oracle, Reference, reference_available

    lib = Reference() if reference_available() else Oracle()
    t0 = time.perf_counter()
    c = lib.decompose(field_np)
    t1 = time.perf_counter()
    lib.recompose(c, field_np.shape)
    t2 = time.perf_counter()
    cpu = {"value": field_np.nbytes / (t2 - t0) / 1e9, "unit": "GB/s", "cores": 1,
           "kind": "reference" if reference_available() else "port",
           "sample": f"one 513^3 f32 decompose ({t1 - t0:.2f} s) + recompose ({t2 - t1:.2f} s), same field, rank 0",
           "cpu": _cpu_model(), "physical_cores": physical_cores()}
    if mg is None:
        return cpu, None
    from oracle.parity import label_flips

    rg = float(field_np.max() - field_np.min())
    mc = mg.decompose(field, h, 0, wsp)
    got = mc.buffer.cpu().numpy()
    par = {"coeff_max_err_over_range": float(np.max(np.abs(got.astype(np.float64) - c))) / rg,
           "coeff_bar": 1e-5, "budget": "tau / 4", "taus": {}}
    for t in (1e-2, 1e-3, 1e-4):
        tau = t * rg
        plan = mg.make_plan(mg.QuantMode.levelwise, tau / 4.0, h)
        s = mg.quantize(mc, plan, wsp)
        lab, _, _ = lib.quantize(c, field_np.shape, plan.bin_widths)
        try:
            n, worst = label_flips(c, s.flat.cpu().numpy(), lab, h.delta_counts(), plan.bin_widths, ulps=1.0)
            ok = True
        except AssertionError as e:
            n, worst, ok = -1, None, str(e)
        rec = mg.recompose(mg.dequantize(s, plan, h, wsp), wsp)
        linf = float((rec - field).abs().max().item())
        par["taus"][f"{t:g}"] = {"label_flips": n, "worst_flip_ulp": worst, "flips_within_1ulp": ok,
                                 "labels": int(lab.size), "linf_over_tau": linf / tau}
    return cpu, par


# --------------------------------------------------------------------- ours

def run_ours(args, ws, rank, local):
    import numpy as np
    import torch

    import paper_2010_05872_b200 as mg
    from synthetic_fields import config2_field

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    esize = 4
    alg_dir, h = hierarchy_bytes(DIMS, esize)
    field = config2_field(DIMS, seed=field_seed(rank), device=dev)
    nbytes = field.numel() * esize
    wsp = mg.SolverWorkspace(device=local, path=args.path)
    stream = torch.cuda.current_stream(dev)

    def step():
        mc = mg.decompose(field, h, 0, wsp)
        return mg.recompose(mc, wsp)

    for _ in range(max(args.warmup, 0)):
        out = step()
    torch.cuda.synchronize()
    err = float((out - field).abs().max().item())
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)

    # eager launches (host enqueues every kernel of the step)
    l0 = wsp.launch_count()
    e0.record(stream)
    for _ in range(args.steps):
        out = step()
    e1.record(stream)
    torch.cuda.synchronize()
    eager_ms = e0.elapsed_time(e1) / args.steps
    launches = (wsp.launch_count() - l0) // max(args.steps, 1)

    # steady state: the step's launch sequence captured once in a CUDA graph
    # (same kernels, same buffers) and replayed; the output must match eager
    graph = None
    if not args.eager:
        side = torch.cuda.Stream(dev)
        side.wait_stream(stream)
        with torch.cuda.stream(side):
            step()
        stream.wait_stream(side)
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            gout = step()
        graph.replay()
        torch.cuda.synchronize()
        if not torch.equal(gout, out):
            raise RuntimeError("graph replay differs from eager execution")
        for _ in range(max(args.warmup, 0)):
            graph.replay()
        torch.cuda.synchronize()

    # decompose and recompose alone, each captured in its own graph (the
    # per-direction GB/s and roofline of SURVEY 8(d))
    dir_graphs = {}
    if not args.eager:
        mc_rec = mg.decompose(field, h, 0, wsp)
        for name, fn in (("decompose", lambda: mg.decompose(field, h, 0, wsp)),
                         ("recompose", lambda: mg.recompose(mc_rec, wsp))):
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                fn()
            g.replay()
            dir_graphs[name] = g
        torch.cuda.synchronize()

    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    barrier(ws)
    torch.cuda.synchronize()
    e0.record(stream)
    for _ in range(args.steps):
        if graph is not None:
            graph.replay()
        else:
            out = step()
    e1.record(stream)
    torch.cuda.synchronize()
    barrier(ws)
    ms = e0.elapsed_time(e1) / args.steps
    dir_ms = {}
    for name, g in dir_graphs.items():
        for _ in range(2):
            g.replay()
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(args.steps):
            g.replay()
        e1.record(stream)
        torch.cuda.synchronize()
        dir_ms[name] = e0.elapsed_time(e1) / args.steps
    clk = clocks.stop()
    ms_max = max_over_ranks(ms, ws)
    value = aggregate_gbs(ws, nbytes, ms_max)
    peak, peak_src = measured_peak()
    step_achieved = 2 * alg_dir / (ms * 1e-3) / 1e9

    # per-kernel device times (CUDA events on the library's stream, keyed
    # "<kernel>@<level>"), decompose and recompose profiled separately over
    # the same number of steps right after the timed region
    mc = mg.decompose(field, h, 0, wsp)
    wsp.profile_begin()
    for _ in range(args.steps):
        mg.decompose(field, h, 0, wsp)
    prof_dec = wsp.profile_end()
    wsp.profile_begin()
    for _ in range(args.steps):
        mg.recompose(mc, wsp)
    prof_rec = wsp.profile_end()
    del mc
    prof = {}
    for src, tagd in ((prof_dec, "dec"), (prof_rec, "rec")):
        for k, (t, n) in src.items():
            key = k if k.split("@")[0] not in ("f3_col0", "f3_col1", "tail_dec", "tail_rec") else f"{k}[{tagd}]"
            prof[key] = (t, n)
    prof_total = sum(v[0] for v in prof.values()) / args.steps
    L = h.num_levels()
    dominant = max(prof.items(), key=lambda kv: kv[1][0]) if prof else ("none", (0.0, 1))
    dom_tag = dominant[0]
    dom_level = int(dom_tag.split("@")[1].split("[")[0]) if "@" in dom_tag else L
    kern_ms = dominant[1][0] / max(dominant[1][1], 1)
    # algorithmic bytes of a level pass: read + write the level block once
    # (2 * s * #N_l); the dominant kernel carries that pass
    kernel_bytes = 2 * esize * h.node_count(dom_level)
    kern_achieved = kernel_bytes / (kern_ms * 1e-3) / 1e9 if kern_ms > 0 else 0.0
    traffic = measured_traffic(dom_tag)
    # finest-level passes: all kernels of level L per direction
    lvl_ms = {}
    for name, src in (("decompose", prof_dec), ("recompose", prof_rec)):
        lvl_ms[name] = sum(t for k, (t, n) in src.items() if k.endswith("@%d" % L)) / args.steps
    lvl_bytes = 2 * esize * h.node_count(L)
    # end-to-end through the host-buffer C-ABI entry points (pinned host
    # memory; H2D of the field + D2H of the coefficients for decompose, H2D
    # of the coefficients + D2H of the field for recompose, every step)
    e2e = e2e_measure(mg, wsp, field, h, args, workers=max(1, args.e2e_workers))
    quant = quant_measure(mg, wsp, field, h, args)
    batch = batch_measure(mg, field, h, args, dev)

    cpu = parity = None
    if rank == 0 and not args.no_cpu_baseline:
        cpu, parity = cpu_baseline_sample(field.cpu().numpy(), mg, wsp, field, h)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": WORKLOAD, "field": list(DIMS), "field_dtype": FIELD_DTYPE,
                       "levels": h.num_levels(), "path": args.path,
                       "l2": f"inputs larger than L2 ({nbytes / 1e6:.0f} MB field vs 126 MB L2); no flush",
                       "parallelism": f"batch: {ws} independent field(s), one per GPU, no collective",
                       "launch": "eager" if graph is None else "cuda_graph (one captured decompose+recompose step, replayed)",
                       "eager_ms_per_step": eager_ms},
            "roofline": {"bound": "hbm", "achieved": step_achieved, "peak": peak, "unit": "GB/s",
                         "frac": step_achieved / peak, "frac_nominal_8tbs": step_achieved / 8000.0,
                         "traffic": step_traffic(), "alg_bytes_per_step": 2 * alg_dir, "peak_source": peak_src,
                         "definition": "the whole step: sum_{l=1..L} 2*s*#N_l per direction (SURVEY 8(d)), "
                                       "decompose + recompose, / device step time; traffic = ncu DRAM read+write "
                                       "bytes of all kernels of one step (profiles/traffic.json)"},
            "directions": {
                k: {"ms": v, "gbs_input": nbytes / (v * 1e-3) / 1e9,
                    "achieved": alg_dir / (v * 1e-3) / 1e9, "frac": alg_dir / (v * 1e-3) / 1e9 / peak,
                    "frac_nominal_8tbs": alg_dir / (v * 1e-3) / 1e9 / 8000.0} for k, v in dir_ms.items()},
            "kernel_roofline": {"bound": "hbm", "achieved": kern_achieved, "peak": peak, "unit": "GB/s",
                                "frac": kern_achieved / peak, "traffic": traffic, "kernel": dom_tag,
                                "kernel_ms": kern_ms, "kernel_alg_bytes": kernel_bytes,
                                "definition": "dominant kernel: 2*s*#N_l of its level / its average CUDA-event "
                                              "duration"},
            "finest_level_roofline": {
                k: {"ms": v, "achieved": lvl_bytes / (v * 1e-3) / 1e9 if v else 0.0,
                    "frac": (lvl_bytes / (v * 1e-3) / 1e9) / peak if v else 0.0} for k, v in lvl_ms.items()},
            "kernels_ms_per_step": {k: v[0] / args.steps for k, v in sorted(prof.items(), key=lambda kv: -kv[1][0])},
            "kernels_launches_per_step": {k: v[1] // args.steps for k, v in prof.items()},
            "profiled_step_ms": prof_total,
            "e2e": e2e,
            "quantize": quant,
            "batch": batch,
            "cpu_baseline": cpu,
            "parity": parity,
            "clocks": clk,
            "gpu_launches": int(launches),
            "roundtrip_linf": err,
        }
        print(json.dumps(line), flush=True)


def step_traffic():
    """ncu DRAM bytes (read + write) of all kernels of one decompose +
    recompose step (profiles/traffic.json "step"), or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            v = json.load(f).get("step")
        return None if v is None else float(v)
    except Exception:
        return None


def measured_traffic(tag):
    """DRAM bytes (read + write) per launch of `tag` from the committed ncu
    launch list summary (profiles/traffic.json), or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            d = json.load(f)
        v = d.get("kernels", {}).get(tag)
        return None if v is None else float(v)
    except Exception:
        return None


def batch_measure(mg, field, h, args, dev, inflight=None):
    """Config 5a on one GPU: independent fields in flight on separate
    streams (one context and one captured step graph each), so one field's
    latency-bound coarse levels overlap another's finest-level passes.
    Reported beside the single-field metric, same bytes per field."""
    import torch

    from synthetic_fields import config2_field

    inflight = inflight or args.batch_inflight
    fields = [field] + [config2_field(DIMS, seed=1000 + i, device=dev) for i in range(inflight - 1)]
    streams = [torch.cuda.Stream(dev) for _ in fields]
    graphs, contexts = [], []  # contexts must outlive the graphs (their scratch is captured)
    for f, st in zip(fields, streams):
        ws = mg.SolverWorkspace(device=dev.index)
        contexts.append(ws)
        st.wait_stream(torch.cuda.current_stream(dev))
        with torch.cuda.stream(st):
            mg.recompose(mg.decompose(f, h, 0, ws), ws)
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=st):
                mg.recompose(mg.decompose(f, h, 0, ws), ws)
        graphs.append(g)
    torch.cuda.synchronize()
    main = torch.cuda.current_stream(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    def run(k):
        for _ in range(k):
            for g, st in zip(graphs, streams):
                st.wait_stream(main)
                with torch.cuda.stream(st):
                    g.replay()
            for st in streams:
                main.wait_stream(st)

    run(2)
    torch.cuda.synchronize()
    k = max(1, args.steps)
    e0.record(main)
    run(k)
    e1.record(main)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / k
    nbytes = sum(f.numel() * f.element_size() for f in fields)
    return {"fields_in_flight": inflight, "ms_per_step": ms, "value": nbytes / (ms * 1e-3) / 1e9, "unit": "GB/s",
            "note": "each step = decompose + recompose of every in-flight field (config 5a style, per GPU)"}


def quant_measure(mg, wsp, field, h, args):
    """Level-wise quantize + dequantize of the step's coefficients (the rest
    of the path, quantize.hpp:39-150) at tau = 1e-3 * range, budget tau / 4;
    device time with CUDA events.  Bytes: N*s + 4N each way."""
    import torch

    mc = mg.decompose(field, h, 0, wsp)
    rg = float((field.max() - field.min()).item())
    plan = mg.make_plan(mg.QuantMode.levelwise, 1e-3 * rg / 4.0, h)
    s = mg.quantize(mc, plan, wsp)
    mg.dequantize(s, plan, h, wsp)
    torch.cuda.synchronize()
    k = max(1, min(args.steps, 10))
    e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
    e0.record()
    for _ in range(k):
        s = mg.quantize(mc, plan, wsp)
    e1.record()
    for _ in range(k):
        d = mg.dequantize(s, plan, h, wsp)
    e2.record()
    torch.cuda.synchronize()
    q_ms, d_ms = e0.elapsed_time(e1) / k, e1.elapsed_time(e2) / k
    nb = field.numel() * (field.element_size() + 4)
    back = mg.recompose(d, wsp)
    linf = float((back - field).abs().max().item())
    # kernel-level device times (library profiler) of one quantize + dequantize
    wsp.profile_begin()
    s = mg.quantize(mc, plan, wsp)
    mg.dequantize(s, plan, h, wsp)
    prof = {kk: v[0] * 1e3 for kk, v in wsp.profile_end().items()}
    # the one-call forms (decompose + quantize, dequantize + recompose) beside the two-call sequences
    def timed(fn):
        fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(k):
            fn()
        b.record()
        torch.cuda.synchronize()
        return a.elapsed_time(b) / k

    one_call = {
        "decompose_then_quantize_ms": timed(lambda: mg.quantize(mg.decompose(field, h, 0, wsp), plan, wsp)),
        "decompose_quantize_ms": timed(lambda: mg.decompose_quantize(field, h, plan, 0, wsp)),
        "dequantize_then_recompose_ms": timed(lambda: mg.recompose(mg.dequantize(s, plan, h, wsp), wsp)),
        "dequantize_recompose_ms": timed(lambda: mg.dequantize_recompose(s, plan, h, wsp)),
        "note": "eager calls; decompose_quantize quantizes the finest shell on a side stream under the rest of "
                "the decomposition",
    }
    peak, _ = measured_peak()
    kern = {}
    for name in ("quant_labels", "dequant"):
        us = prof.get(name)
        if us:
            kern[name] = {"us": us, "achieved_gbs": nb / (us * 1e-6) / 1e9, "frac": nb / (us * 1e-6) / 1e9 / peak}
    return {"quantize_ms": q_ms, "dequantize_ms": d_ms, "quantize_gbs": nb / (q_ms * 1e-3) / 1e9,
            "dequantize_gbs": nb / (d_ms * 1e-3) / 1e9, "quantize_frac": nb / (q_ms * 1e-3) / 1e9 / peak,
            "dequantize_frac": nb / (d_ms * 1e-3) / 1e9 / peak, "kernels_us": prof, "kernel_roofline": kern,
            "alg_bytes": nb, "outliers": int(s.outlier_positions.numel()), "one_call": one_call,
            "linf_over_tau": linf / (1e-3 * rg), "tau": "1e-3 * range, budget tau/4",
            "note": "whole calls include the outlier-count readback (synchronous, as the reference's API); "
                    "bytes N*s + 4N each way (SURVEY 8(d))"}


def e2e_measure(mg, wsp, field, h, args, workers=2):
    """Same metric through the host-buffer C-ABI (mgrx_host_decompose +
    mgrx_host_recompose; every step copies its field H2D from pinned memory,
    its coefficients D2H and back, and its reconstruction D2H).  `workers`
    host threads, one context (stream) each, so one step's copies overlap
    the next step's copies in the other direction (both copy engines busy)."""
    import ctypes as C
    import threading

    import torch

    from paper_2010_05872_b200._lib import lib

    dims = (C.c_uint64 * len(DIMS))(*DIMS)
    nbytes = field.numel() * field.element_size()
    dt_code = 0 if field.dtype == torch.float32 else 1
    ctxs, bufs = [], []
    for w in range(workers):
        ctx = wsp if w == 0 else mg.SolverWorkspace(device=field.device.index)
        host_in = field.cpu().pin_memory()
        host_c = torch.empty(field.numel(), dtype=field.dtype).pin_memory()
        host_out = torch.empty_like(host_in).pin_memory()
        ctxs.append(ctx)
        bufs.append((host_in, host_c, host_out))

    def one(w):
        host_in, host_c, host_out = bufs[w]
        rc = lib.mgrx_host_decompose(ctxs[w].handle, dt_code, len(DIMS), dims, -1, 0, C.c_void_p(host_in.data_ptr()),
                                     C.c_void_p(host_c.data_ptr()))
        assert rc == 0, rc
        rc = lib.mgrx_host_recompose(ctxs[w].handle, dt_code, len(DIMS), dims, -1, 0, C.c_void_p(host_c.data_ptr()),
                                     C.c_void_p(host_out.data_ptr()))
        assert rc == 0, rc

    for w in range(workers):
        one(w)
    k = max(workers, min(args.steps, 6))
    per = [k // workers + (1 if w < k % workers else 0) for w in range(workers)]

    def run(w):
        for _ in range(per[w]):
            one(w)

    t0 = time.perf_counter()
    ts = [threading.Thread(target=run, args=(w,)) for w in range(workers)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    dt = (time.perf_counter() - t0) / k
    err = float((bufs[0][2].to(field.device) - field).abs().max().item())
    return {"value": nbytes / dt / 1e9, "unit": "GB/s", "h2d_bytes_per_step": 2 * nbytes,
            "d2h_bytes_per_step": 2 * nbytes, "ms_per_step": dt * 1e3, "steps": k, "roundtrip_linf": err,
            "path": f"mgrx_host_decompose + mgrx_host_recompose (pinned host buffers), {workers} host threads "
                    "with one context each (copies of consecutive steps overlap)"}


def run_slab(args, ws, rank, local):
    """Slab mode: ONE field split into axis-0 slabs over the ws
    ranks (paper_2010_05872_b200/slab.py: halo exchange + NCCL all-to-all
    transposes for the axis-0 solve).  Strong scaling: value = the whole
    field's bytes / the slowest rank's step time.  With ws == 1 and
    --slab-emulate R > 1, all R ranks run on this one GPU with device copies
    for the exchanges (a correctness / overhead check: the time is the SUM
    over the emulated ranks, not a multi-GPU number)."""
    import torch

    import paper_2010_05872_b200 as mg
    from synthetic_fields import config2_field
    from paper_2010_05872_b200.slab import LocalExchange, PlaneSlab, TorchExchange, max_slab_levels, \
        owned_planes, slab_bounds, slab_decompose, slab_recompose

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    field = config2_field(DIMS, seed=0, device=dev)
    h = mg.GridHierarchy.create(DIMS)
    emul = ws == 1 and args.slab_emulate > 1
    ex = LocalExchange(args.slab_emulate) if emul else (TorchExchange() if ws > 1 else LocalExchange(1))
    R = ex.world
    S = max_slab_levels(h, R)
    P = slab_bounds(DIMS[0], R, S)
    plane = DIMS[1] * DIMS[2]
    fields = []
    for r in ex.local:  # each rank holds only its own planes
        lo, hi = owned_planes(P, r, DIMS[0])
        s = PlaneSlab(lo, hi, plane, field.dtype, dev)
        s.t.copy_(field.reshape(DIMS[0], -1)[lo:hi])
        fields.append(s)
    wss = [mg.SolverWorkspace(device=local) for _ in ex.local]
    stream = torch.cuda.current_stream(dev)

    def step():
        outs = slab_decompose(fields, h, ex, wss, S)
        return slab_recompose(outs, h, ex, wss), outs

    for _ in range(max(args.warmup, 1)):
        backs, outs = step()
    torch.cuda.synchronize()
    err = 0.0
    fv = field.reshape(DIMS[0], -1)
    for i, r in enumerate(ex.local):
        lo, hi = owned_planes(P, r, DIMS[0])
        d = (backs[i].planes(lo, hi) - fv[lo:hi]).abs()
        err = max(err, float("inf") if bool(torch.isnan(d).any()) else float(d.max().item()))
    rank_bytes = max(o.nbytes() for o in outs)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier(ws)
    torch.cuda.synchronize()
    e0.record(stream)
    for _ in range(args.steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    ms = max_over_ranks(e0.elapsed_time(e1) / args.steps, ws, device=dev)
    nbytes = field.numel() * 4
    if rank == 0:
        line = {"metric": METRIC, "value": nbytes / (ms * 1e-3) / 1e9, "unit": "GB/s", "n_gpus": ws,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": {"workload": WORKLOAD + " -- slab mode (one field split along axis 0)",
                           "field": list(DIMS), "field_dtype": "f32", "ranks": R, "slab_levels": S,
                           "slab_bounds": P, "emulated_on_one_gpu": emul,
                           "coefficient_bytes_per_rank": rank_bytes,
                           "parallelism": f"slab{R}" + (" (emulated: time is the sum over ranks)" if emul else "")},
                "roundtrip_linf": err}
        print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--path", choices=["auto", "general"], default="auto")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--eager", action="store_true", help="time eager launches instead of CUDA-graph replay")
    ap.add_argument("--batch-inflight", type=int, default=2, help="fields in flight for the batch measurement")
    ap.add_argument("--dims", default="513,513,513",
                    help="field extents (config-2 generator); 1025,1025,1025 is BASELINE config 5b")
    ap.add_argument("--ref-threads", type=int, default=0)
    ap.add_argument("--warmup-ref", type=int, default=0, help="untimed reference steps (CPU code needs none)")
    ap.add_argument("--e2e-workers", type=int, default=2, help="host threads (contexts) of the e2e measurement")
    ap.add_argument("--slab", action="store_true",
                    help="slab mode: one field split along axis 0 over the ranks (NCCL transposes); strong scaling")
    ap.add_argument("--slab-emulate", type=int, default=1,
                    help="with --slab on one GPU: emulate this many ranks in-process (correctness/overhead check)")
    ap.add_argument("--dist-selftest", action="store_true", help=argparse.SUPPRESS)
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(self_launch(args.gpus, sys.argv[1:]))
    if "WORLD_SIZE" in os.environ and args.impl == "ours" and not args.dist_selftest:
        wsz = int(os.environ["WORLD_SIZE"])
        if wsz != args.gpus:
            print(f"[bench] note: --gpus {args.gpus} but WORLD_SIZE {wsz}; using WORLD_SIZE", file=sys.stderr)
    if args.dist_selftest:
        dist_selftest(args)
        return
    global DIMS, WORKLOAD
    dims = tuple(int(x) for x in args.dims.split(","))
    if dims != DIMS:
        DIMS = dims
        tag = "config5b" if dims == (1025, 1025, 1025) else "config2-generator"
        WORKLOAD = (f"{tag}: {'x'.join(map(str, dims))} fp32 field (16 bumps + 8 oblique sine modes + 1e-4 noise), "
                    "full decompose + recompose (stop 0)")
    if args.impl == "reference":
        # rank 0 alone runs the CPU reference; other torchrun ranks exit 0
        run_reference(args, int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")))
        return
    ws, rank, local = dist_init()
    if args.slab:
        run_slab(args, ws, rank, local)
    else:
        run_ours(args, ws, rank, local)
    if ws > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


if __name__ == "__main__":
    main()
