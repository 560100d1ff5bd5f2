#!/usr/bin/env python3
"""PAGANI hot-path benchmark (contract: one JSON line on rank 0).

Workload (BASELINE.json configs[1]): the 8D Genz suite f1..f6 at
epsrel in {1e-3, 1e-4, 1e-5, 1e-6}, tau_abs=1e-20, it_max=100,
max_regions=2^22 (the reference defaults), relative filtering off for f1 only
(bfcub_cli.cpp:77-78).  One "step" = the 24 integrate() calls.

  value   region-evals/s over the step, device time: the CUDA-event span of
          each integrate() on the library's stream (inputs: none -- the
          region list is generated and kept in HBM by the library)
  e2e     the same metric through the public Python API / C ABI, host wall
          clock, including every host<->device copy (bounds/config in, the
          per-iteration scalar read-backs and the result out)
  roofline  k_evaluate (FP64 CUDA-core bound): algorithmic FLOPs
          (paper_2104_06494_b200/roofline.py) / its summed
          CUDA-event time, against an FP64 DFMA peak measured live on the box
  cpu_baseline  the unmodified reference library (oracle/_ref) on the box's
          host cores on a bounded sample of the same workload

--impl reference runs that reference library (all host threads) on the
bounded sample for every step.  Multi-GPU (torchrun): the region list of every
integrate() is sharded over the ranks (NCCL; strong scaling) -- DESIGN.md §7.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "time-to-tolerance (s) & region-evals/s, 8D Genz f1–f6, at 1/2/4/8 B200"
UNIT = "region-evals/s"
DIM = 8
TAUS = (1e-3, 1e-4, 1e-5, 1e-6)
FIDS = (1, 2, 3, 4, 5, 6)
# Bounded CPU sample of the same workload: a faithful subset of the suite --
# three of its 24 integrate() calls, run to their end exactly as in the suite
# (same config, same outcome), ~6 s of reference CPU time per step on 16 cores
# (so --steps 20 --warmup 5 of the reference arm takes ~2.5 minutes).  The GPU
# arm runs the same two calls inside its timed steps and reports its rate on
# them ("same_sample"), so the GPU/CPU ratio on identical work is derivable.
CPU_SAMPLE = ((3, 1e-3), (3, 1e-4), (5, 1e-3))
CPU_SAMPLE_DESC = ("complete integrate() calls f3@1e-3, f3@1e-4, f5@1e-3 (8D, suite config: "
                   "3 of the suite's 24 cases, run to their end; 15.2M region-evals)")
# 1-thread protocol run: one call of the sample
CPU_SAMPLE_1T = ((3, 1e-4),)


def dist_env():
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def workload(cases=None):
    """All (fid, tau) of the suite, or a subset like "f4@1e-3,f1@1e-3"."""
    if cases:
        out = []
        for c in cases.split(","):
            f, t = c.split("@")
            out.append((int(f.strip().lstrip("f")), float(t)))
        return out
    return [(fid, tau) for fid in FIDS for tau in TAUS]


# ----------------------------------------------------------------- clocks ---
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.proc = None
        self.path = None

    def start(self):
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        rows = []
        for line in open(self.path):
            p = [x.strip() for x in line.split(",")]
            if len(p) < 9:
                continue
            try:
                rows.append((float(p[1]), float(p[2]), p[5:9]))
            except ValueError:
                continue
        os.unlink(self.path)
        if not rows:
            return None
        sm_max = max(r[1] for r in rows)
        loaded = [r for r in rows if r[0] > 0.3 * sm_max] or rows
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i, v in enumerate(r[2]) if v == "Active"})
        return {"sm_mhz": statistics.median(r[0] for r in loaded), "sm_max_mhz": sm_max,
                "reasons": reasons, "samples": len(rows)}


def measured_hbm_peak():
    """HBM copy bandwidth from the driver-written MEASURED_PEAKS.json (GB/s)."""
    try:
        d = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        return float(d["hbm_gbs"]), "of measured: MEASURED_PEAKS.json hbm_gbs (copy bandwidth)"
    except Exception:  # noqa: BLE001
        return 6650.0, "of fallback: 6.65 TB/s (B200_PROFILING.md; MEASURED_PEAKS.json absent)"


def bench_config(args):
    """The workload's config, identical in both arms (the reference arm times a
    bounded sample of this same workload; its cpu_baseline.sample says which)."""
    return {"workload": "genz_8d_suite: f1..f6 x tau in {1e-3,1e-4,1e-5,1e-6}, n=8, "
                        "tau_abs=1e-20, it_max=100, rel filter off for f1",
            "max_regions": args.max_regions, "mode": args.mode,
            "l2": "working set > L2: each run streams a region store of up to 1.1 GB"}


try:  # before any OpenMP runtime binds this thread (OMP_PROC_BIND shrinks the mask)
    _USABLE_CPUS = len(os.sched_getaffinity(0))
except Exception:  # noqa: BLE001
    _USABLE_CPUS = os.cpu_count()


def host_cpu():
    """CPU model and core counts from lscpu."""
    info = {"model": None, "sockets": 1, "cores_per_socket": None, "threads_per_core": 1,
            "logical": os.cpu_count()}
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        kv = {}
        for line in out.splitlines():
            if ":" in line:
                k, v = line.split(":", 1)
                kv[k.strip()] = v.strip()
        info["model"] = kv.get("Model name")
        info["sockets"] = int(kv.get("Socket(s)", "1") or 1)
        info["cores_per_socket"] = int(kv.get("Core(s) per socket", "0") or 0) or None
        info["threads_per_core"] = int(kv.get("Thread(s) per core", "1") or 1)
    except Exception:  # noqa: BLE001
        pass
    if info["cores_per_socket"]:
        info["physical"] = info["sockets"] * info["cores_per_socket"]
    else:
        info["physical"] = max(1, (os.cpu_count() or 1) // max(1, info["threads_per_core"]))
    info["usable"] = _USABLE_CPUS
    return info


def load_reference():
    """The unmodified reference (oracle/_ref).  OpenMP placement must be in the
    environment before libgomp initialises, i.e. before the library loads."""
    os.environ.setdefault("OMP_PROC_BIND", "close")
    os.environ.setdefault("OMP_PLACES", "cores")
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from ref_ctypes import Ref, make_config
    return Ref(), make_config


def comm_info(args, world, comm, rank_clocks):
    """What the ranks ran over (checkable against NCCL_DEBUG=INFO logs)."""
    info = {"world_size": world, "sharded": comm is not None,
            "comm_nranks": getattr(comm, "size", 1) if comm is not None else 1}
    if world > 1:
        info["backend"] = args.dist_backend
        try:
            import torch
            info["nccl_version"] = ".".join(str(v) for v in torch.cuda.nccl.version())
        except Exception:  # noqa: BLE001
            pass
        info["per_rank_clocks"] = rank_clocks
    return info


# --------------------------------------------------------------- ours -------
def run_ours(args, rank, world, local_rank):
    import paper_2104_06494_b200 as pg
    from paper_2104_06494_b200 import roofline

    torch = None
    comm = None
    parallelism = "1 GPU"
    if world > 1:
        import torch
        import torch.distributed as dist
        local_rank = local_rank % max(1, torch.cuda.device_count())
        torch.cuda.set_device(local_rank)
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        else:  # gloo host transport: lets several ranks share one GPU (testing)
            dist.init_process_group("gloo")
        from paper_2104_06494_b200 import dist as pdist
        try:  # sharded: one region list split over the ranks (strong scaling)
            comm = pdist.from_torch(local_rank)
            parallelism = (f"sharded over {world} ranks ({args.dist_backend}: allgather of block "
                           f"records + send/recv exchange, DESIGN.md 7)")
        except Exception as e:  # noqa: BLE001 - still GPU work, just not sharded
            comm = None
            parallelism = f"replicas x{world} (sharding unavailable: {e})"
    device = local_rank

    def barrier_sync():
        if world > 1:
            torch.distributed.barrier()
            torch.cuda.synchronize()

    def _reduce(x, op):
        if world == 1:
            return x
        dev = "cuda" if args.dist_backend == "nccl" else "cpu"
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        torch.distributed.all_reduce(t, op=op)
        return float(t.item())

    def max_over_ranks(x):
        return _reduce(x, torch.distributed.ReduceOp.MAX) if world > 1 else x

    def sum_over_ranks(x):
        return _reduce(x, torch.distributed.ReduceOp.SUM) if world > 1 else x

    mode = args.mode
    cases = workload(args.cases)

    call_wall = {}  # (fid, tau) -> host wall seconds of each timed call

    def one_step(profile, timed=False):
        rs = []
        for fid, tau in cases:
            cfg = pg.Config(tau_rel=tau, rel_filtering_enabled=(fid != 1), max_regions=args.max_regions,
                            mode=mode, device=device, profile=profile, comm=comm)
            t0 = time.perf_counter()
            r = pg.integrate(pg.Integrand(fid), pg.Bounds.unit_cube(DIM), cfg)
            if timed:
                call_wall[(fid, tau)] = call_wall.get((fid, tau), 0.0) + time.perf_counter() - t0
            rs.append((fid, tau, r))
        return rs

    # Timed steps record CUDA events around k_evaluate only (profile=2): the
    # event-record calls of a fully instrumented step sit on the host's side
    # of every host-decision gap and cost ~2% of the step (measured: 2021 vs
    # 2062-2072 ms).  The other kernel classes' times (hbm_rooflines,
    # kernel_ms_per_step) come from one fully instrumented step (profile=1)
    # run after the timed region on the same workload.
    for _ in range(args.warmup):
        one_step(2)

    peak_tflops, peak_mhz = pg.api.fp64_peak(device, 1.0)

    clocks = ClockSampler(int(os.environ.get("CUDA_VISIBLE_DEVICES", str(device)).split(",")[0])
                          if os.environ.get("CUDA_VISIBLE_DEVICES", "").isdigit() else device)
    clocks.start()
    barrier_sync()
    t_wall0 = time.perf_counter()
    steps = []
    for _ in range(args.steps):
        steps.append(one_step(2, timed=True))
    barrier_sync()
    t_wall = time.perf_counter() - t_wall0
    clk = clocks.stop()
    inst_step = one_step(1)  # per-kernel breakdown, outside the timed region
    rank_clocks = [clk]
    if world > 1:  # every rank's clocks (max-over-ranks timing needs all of them sane)
        rank_clocks = [None] * world
        torch.distributed.all_gather_object(rank_clocks, clk)

    dev_ms = sum(r.device_ms for st in steps for _, _, r in st)
    region_evals = sum(r.region_evals for st in steps for _, _, r in st)
    eval_ms = sum(r.kernel_ms["evaluate"] for st in steps for _, _, r in st)
    eval_launches = sum(r.kernel_launches["evaluate"] for st in steps for _, _, r in st)
    flops = sum(r.region_evals * roofline.region_flops(fid, DIM) for st in steps
                for fid, _, r in st)
    launches = sum(sum(r.kernel_launches.values()) for st in steps for _, _, r in st)
    h2d = sum(r.h2d_bytes for st in steps for _, _, r in st) / args.steps
    d2h = sum(r.d2h_bytes for st in steps for _, _, r in st) / args.steps

    # e2e: the public API's host wall clock over the same K steps
    dev_s_max = max_over_ranks(dev_ms / 1e3)
    wall_s_max = max_over_ranks(t_wall)
    evals_all = sum_over_ranks(region_evals)
    value = evals_all / dev_s_max
    e2e_value = evals_all / wall_s_max

    if rank != 0:
        return
    per_case = []
    import importlib
    suite = importlib.import_module("paper_2104_06494_b200.suite")  # the module, not pg.suite()
    for fid, tau, r in steps[-1]:
        exact = suite.reference_value(f"f{fid}", DIM, corrected=True)
        true_rel = abs(r.estimate - exact) / abs(exact) if exact else None
        per_case.append({"f": f"f{fid}", "tau": tau, "status": str(r.status),
                         "it": r.iterations, "regions": r.regions_generated,
                         "estimate": r.estimate, "errorest": r.errorest,
                         "true_rel_err": true_rel,
                         "true_rel_err_le_tau": bool(true_rel is not None and true_rel <= tau),
                         "time_to_result_s": r.device_ms / 1e3})
    achieved = flops / (eval_ms / 1e3) / 1e12 if eval_ms > 0 else 0.0
    # per integrand: the algorithmic count is the reference's arithmetic, so an
    # integrand whose per-point work the separable evaluator shares (f2: the n
    # divisions per point become 9n per region) can exceed the peak; ncu's
    # FP64-pipe utilisation is the executed-work view.
    per_f = {}
    for fid in sorted({f for f, _ in cases}):
        ms = sum(r.kernel_ms["evaluate"] for st in steps for f, _, r in st if f == fid)
        fl = sum(r.region_evals * roofline.region_flops(f, DIM) for st in steps
                 for f, _, r in st if f == fid)
        if ms > 0:
            per_f[f"f{fid}"] = round(fl / (ms / 1e3) / 1e12, 2)
    # HBM rooflines of the memory-side kernels: algorithmic bytes (DESIGN.md 4,
    # counted by the driver per launch) / their CUDA-event time.
    hbm_peak, hbm_src = measured_hbm_peak()
    hbm = {}
    split_label = ("k_split (filter + bisect)" if os.environ.get("PAGANI_DEFER_BISECT") == "0"
                   else "k_link (filter; the bisection is deferred into k_evaluate, DESIGN.md 4)")
    for k, label in (("split", split_label),
                     ("probe", "k_probe_multi + trees (threshold classify)")):
        ms = sum(r.kernel_ms[k] for _, _, r in inst_step)
        by = sum(r.kernel_bytes[k] for _, _, r in inst_step)
        if ms > 0:
            gbs = by / (ms / 1e3) / 1e9
            hbm[k] = {"kernel": label, "achieved": gbs, "peak": hbm_peak, "unit": "GB/s",
                      "frac": gbs / hbm_peak if hbm_peak else None,
                      "bytes_per_step": by, "ms_per_step": ms,
                      "measured_on": "one fully instrumented step after the timed region"}
    # executed-work view: ncu-counted FP64 operations per region-evaluation
    # (2 per DFMA, 1 per DMUL / DADD; profiles/r02_executed_flops.json) times
    # this run's region-evaluations over its CUDA-event time
    executed = None
    try:
        ex = json.load(open(os.path.join(ROOT, "profiles", "r02_executed_flops.json")))
        per = ex["per_integrand"]
        ex_fl, ex_per_f = 0.0, {}
        for fid in sorted({f for f, _ in cases}):
            k = f"f{fid}"
            if k not in per:
                continue
            ev = sum(r.region_evals for st in steps for f, _, r in st if f == fid)
            ms = sum(r.kernel_ms["evaluate"] for st in steps for f, _, r in st if f == fid)
            fl = ev * per[k]["executed_fp64_flops_per_region"]
            ex_fl += fl
            if ms > 0:
                ex_per_f[k] = round(fl / (ms / 1e3) / 1e12, 2)
        if eval_ms > 0 and ex_fl > 0:
            ex_t = ex_fl / (eval_ms / 1e3) / 1e12
            executed = {"tflops": ex_t, "frac": ex_t / peak_tflops if peak_tflops else None,
                        "tflops_per_integrand": ex_per_f,
                        "note": "FP64 ops the kernel executes (ncu SASS op counters per region-"
                                "evaluation, 8D, profiles/r02_executed_flops.json) x this run's "
                                "region-evaluations / k_evaluate time; fewer than the reference's "
                                "arithmetic (shared separable terms) and mostly DADD/DMUL (parity "
                                "forbids fusing), so the DFMA-rate peak is out of reach by design"}
    except Exception:  # noqa: BLE001
        executed = None
    traffic = None
    prof_path = os.path.join(ROOT, "profiles", "ncu_evaluate_summary.json")
    if os.path.exists(prof_path):
        try:
            traffic = json.load(open(prof_path)).get("dram_bytes_per_launch")
        except Exception:
            traffic = None
    # the GPU's rate on exactly the reference arm's sample (same calls, taken
    # from the timed steps above)
    same = None
    samp = [c for c in CPU_SAMPLE if c in set(cases)]
    if samp:
        ev = sum(r.region_evals for st in steps for f, t, r in st if (f, t) in samp)
        ms = sum(r.device_ms for st in steps for f, t, r in st if (f, t) in samp)
        wall = sum(call_wall.get(c, 0.0) for c in samp)
        same = {"sample": CPU_SAMPLE_DESC, "value": ev / (ms / 1e3) if ms else None,
                "e2e_value": ev / wall if wall else None, "unit": UNIT,
                "region_evals_per_step": ev // args.steps,
                "ms_per_step": ms / args.steps}
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline()
        if same and cpu.get("value"):
            same["vs_cpu_baseline"] = same["value"] / cpu["value"]
            same["e2e_vs_cpu_baseline"] = (same["e2e_value"] or 0.0) / cpu["value"]
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": dev_s_max * 1e3 / args.steps,
        "higher_is_better": True, "scaling": "strong" if comm is not None or world == 1 else "weak",
        "vs_baseline": None, "dtype": "f64",
        "data": "synthetic: the reference's fixed-parameter Genz integrands (deterministic, no dataset)",
        "config": bench_config(args),
        "parallelism": parallelism,
        "roofline": {"bound": "fp64", "kernel": "k_evaluate_sep", "achieved": achieved,
                     "peak": peak_tflops, "unit": "TFLOP/s",
                     "frac": achieved / peak_tflops if peak_tflops else None,
                     "traffic": traffic,
                     "peak_source": f"measured live: DFMA microbenchmark (pagani_fp64_peak) at "
                                    f"{peak_mhz:.0f} MHz; MEASURED_PEAKS.json has no FP64 entry",
                     "flops_model": "SURVEY.md 8(d) F(f,n), paper_2104_06494_b200/roofline.py",
                     "tflops_per_integrand": per_f,
                     "executed": executed,
                     "eval_ms": eval_ms / args.steps, "eval_launches": eval_launches // args.steps,
                     "eval_share_of_step": eval_ms / dev_ms if dev_ms else None,
                     "kernel_ms_per_step": {k: round(sum(r.kernel_ms[k] for _, _, r in inst_step), 3)
                                            for k in ("evaluate", "fold", "finalize", "minmax",
                                                      "probe", "split", "init")},
                     "kernel_ms_per_step_note": "one fully instrumented step (profile=1) after "
                                                "the timed region; the timed steps record events "
                                                "around k_evaluate only (profile=2)",
                     "instrumented_step_ms": sum(r.device_ms for _, _, r in inst_step)},
        "hbm_rooflines": {"peak_source": hbm_src, **hbm},
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": int(h2d),
                "d2h_bytes_per_step": int(d2h)},
        "gpu_launches": launches,
        "clocks": clk,
        "comm": comm_info(args, world, comm, rank_clocks),
        "same_sample": same,
        "time_to_tolerance_s": {f"{c['f']}@{c['tau']:g}": round(c["time_to_result_s"], 6)
                                for c in per_case},
        "outcomes": per_case,
    }
    if cpu is not None:
        line["cpu_baseline"] = cpu
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------- reference --
def ref_sample(ref, make_config, threads, cases=CPU_SAMPLE):
    """One bounded sample of the workload on the reference library: complete
    integrate() calls of suite cases (suite config), timed with a steady clock
    around each call as the reference CLI does (bfcub_cli.cpp:81-83)."""
    evals = 0
    secs = 0.0
    for fid, tau in cases:
        # Config::threads -> omp_set_num_threads (driver.cpp); torchrun exports
        # OMP_NUM_THREADS=1 to its workers, so it is set explicitly
        cfg = make_config(tau_rel=tau, rel_filtering_enabled=(fid != 1), threads=threads)
        t0 = time.perf_counter()
        r = ref.integrate(fid, DIM, cfg)
        secs += time.perf_counter() - t0
        evals += r.eval_count // ((1 << DIM) + 2 * DIM * (DIM - 1) + 4 * DIM + 1)
    return evals, secs


def cpu_desc(cpu, threads):
    return (f"{cpu['model']}: {cpu['physical']} physical cores ({cpu['sockets']} socket(s) x "
            f"{cpu['cores_per_socket']} cores x {cpu['threads_per_core']} threads/core, "
            f"{cpu['logical']} logical, {cpu['usable']} usable); OpenMP threads = {threads}, "
            f"OMP_PROC_BIND={os.environ.get('OMP_PROC_BIND')} OMP_PLACES={os.environ.get('OMP_PLACES')}")


def one_thread_rate(ref, make_config):
    e, s = ref_sample(ref, make_config, 1, CPU_SAMPLE_1T)
    return {"value": e / s, "unit": UNIT, "threads": 1,
            "sample": "complete integrate() call f3@1e-4 (8D, suite config)",
            "region_evals": e, "seconds": round(s, 3)}


def cpu_baseline():
    """The reference on the box's host cores: the bounded sample with every
    usable core (median of 3, the runs are < 60 s) and the 1-thread rate."""
    cpu = host_cpu()
    threads = cpu["usable"] or cpu["logical"] or 1
    ref, make_config = load_reference()
    runs = [ref_sample(ref, make_config, threads) for _ in range(3)]
    evals, secs = sorted(runs, key=lambda r: r[1])[1]
    return {"value": evals / secs, "unit": UNIT, "cores": threads, "kind": "reference",
            "sample": CPU_SAMPLE_DESC + f"; {evals} region-evals in {secs:.2f} s (median of 3)",
            "host": cpu_desc(cpu, threads), "cpu_model": cpu["model"],
            "physical_cores": cpu["physical"], "logical_cpus": cpu["logical"],
            "one_thread": one_thread_rate(ref, make_config)}


def run_reference(args, rank, world):
    if rank != 0:
        return
    cpu = host_cpu()
    threads = cpu["usable"] or cpu["logical"] or 1
    try:
        ref, make_config = load_reference()
    except Exception as e:  # the reference is compiled in-tree; this should not happen
        print(json.dumps({"impl": "reference", "unavailable": f"oracle/_ref not loadable: {e}"}))
        return
    for _ in range(args.warmup):
        ref_sample(ref, make_config, threads)
    tot_e, tot_s = 0, 0.0
    for _ in range(args.steps):
        e, s = ref_sample(ref, make_config, threads)
        tot_e += e
        tot_s += s
    value = tot_e / tot_s
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot_s / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic: the reference's fixed-parameter Genz integrands (deterministic)",
        "config": bench_config(args),
        "parallelism": "reference CPU (bfcub, OpenMP), rank 0 only",
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "reference",
                         "sample": CPU_SAMPLE_DESC, "host": cpu_desc(cpu, threads),
                         "cpu_model": cpu["model"], "physical_cores": cpu["physical"],
                         "logical_cpus": cpu["logical"],
                         "one_thread": one_thread_rate(ref, make_config)},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def relaunch_distributed(args):
    """`bench.py --gpus N` (N > 1) outside torchrun: start the N ranks here,
    one process per GPU, exactly as the driver's torchrun command does."""
    import torch
    have = torch.cuda.device_count()
    if have < args.gpus and not (args.dist_backend == "gloo" and have >= 1):
        print(json.dumps({"error": f"--gpus {args.gpus} requested but only {have} GPU(s) visible"}),
              flush=True)
        sys.exit(2)
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1", f"--master-port={port}",
           os.path.abspath(__file__)] + sys.argv[1:]
    os.execv(sys.executable, cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--mode", default="parity", choices=["parity", "fast"])
    ap.add_argument("--max-regions", type=int, default=1 << 22)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="gloo = host transport, for running several ranks on one GPU")
    ap.add_argument("--cases", default=None,
                    help="profiling subset, e.g. f4@1e-3 (the default is the whole suite)")
    args = ap.parse_args()
    rank, world, local_rank = dist_env()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        relaunch_distributed(args)  # does not return
    if args.impl == "ours" and world != args.gpus:
        print(json.dumps({"error": f"--gpus {args.gpus} but WORLD_SIZE={world}: launch one rank "
                                   f"per GPU (torchrun --nproc-per-node {args.gpus})"}), flush=True)
        sys.exit(2)
    if args.impl == "reference":
        run_reference(args, rank, world)
    else:
        run_ours(args, rank, world, local_rank)


if __name__ == "__main__":
    main()
