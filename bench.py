#!/usr/bin/env python
"""bench.py -- triangle-count |E|/s of the block-based TC path on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--impl ours|reference]

One step = one pgabb_triangle_count over the whole graph (S9..S11: the block
intersections of every task this rank owns, the count reduction and, for N>1,
the 8-byte NCCL allreduce), with the block CSR already resident in HBM.  Build
(S1..S8) is pre-processing, excluded as in the paper and
reported separately.  `e2e` is the same metric through the same public call on
a host-resident handle: every step copies the blocks host->device from pinned
memory and reads the count back (the paper's own protocol).

Rank 0 prints ONE JSON line.  See DESIGN.md §6 for every field.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "triangle-count edges/sec (|E|/time)"
UNIT = "edges/s"


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1,
                    help="GPUs (= ranks, one process per GPU).  Without WORLD_SIZE in the environment "
                         "bench.py relaunches itself under torch.distributed.run with N ranks")
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default="c5",
                    help="c5 (Graph500 R-MAT s26 ef32, the headline) | c2 | c3 | c4 | c1 | c5s")
    ap.add_argument("--p", type=int, default=0, help="override parts per dimension")
    ap.add_argument("--cut-rule", type=int, default=0)
    ap.add_argument("--orient", default="auto", choices=["auto", "low", "mid"],
                    help="task orientation (DESIGN R25): per task the one streaming fewer ids, or all LOW / MID")
    ap.add_argument("--light-held", type=int, default=0, choices=[0, 8, 15],
                    help="thread-per-row items up to 8 or 15 held ids (DESIGN R29); 0 = auto")
    ap.add_argument("--path", choices=["count", "vertex", "vertex2", "cc"], default="count",
                    # vertex2: the two-pass route of R24 (measured far slower: kept for the record)
                    help="count: T (the headline); vertex: per-vertex t(v) (SURVEY 8(f) NEXT-1); "
                         "cc: Shiloach-Vishkin connected components on the same blocks (NEXT-4)")
    ap.add_argument("--balance", choices=["measured", "cost"], default="measured",
                    help="N>1: plan pieces with measured task times (R22) or the S7 cost (R17)")
    ap.add_argument("--budget-gb", type=float, default=0.0,
                    help="> 0: blocks stay in pinned host memory and each count streams them through "
                         "a device budget of this many GB (S9 out-of-core mode, PAPER.md:829-835)")
    ap.add_argument("--host-permille", type=int, default=0,
                    help="> 0: collaborative CPU + GPU (NEXT-3) -- blocks in pinned host memory, the "
                         "sparsest pieces up to this share of the cost counted by host threads")
    ap.add_argument("--shared-gpu", action="store_true",
                    help="flow tests only: allow more ranks than visible GPUs (ranks share a GPU, gloo)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--cpu-seconds", type=float, default=15.0, help="target oracle sample time")
    return ap.parse_args(argv)


def self_launch(args):
    """--gpus N without a torchrun environment: check that N GPUs are visible and
    re-run this script as N ranks (one process per GPU) under torch.distributed.run."""
    import socket
    import torch
    ndev = torch.cuda.device_count()
    if ndev < args.gpus and not args.shared_gpu:
        print(json.dumps({"metric": METRIC, "error": f"--gpus {args.gpus} but only {ndev} CUDA device(s) visible"}),
              flush=True)
        sys.exit(1)
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
    sys.exit(subprocess.call(cmd))


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def load_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            pk = json.load(f)
        return float(pk["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


NOMINAL_HBM_GBS = 8000.0   # the north star's ~8 TB/s nominal B200 HBM3e figure (the stricter denominator)
KERNEL_SOURCES = ("paper_2209_04541_b200/csrc/count.cu", "paper_2209_04541_b200/csrc/internal.h")


def kernel_src_hash():
    """sha256 (12 hex) of the S10 kernel sources: an ncu summary is current only for this hash."""
    import hashlib
    h = hashlib.sha256()
    for f in KERNEL_SOURCES:
        with open(os.path.join(ROOT, f), "rb") as fh:
            h.update(fh.read())
    return h.hexdigest()[:12]


def ncu_entry(config, kernel):
    """The committed ncu capture of `kernel` on `config` (profiles/ncu_summary.json,
    written by tools/make_profile.py from an `ncu --set full` / counter capture of this
    command on a B200): DRAM bytes per launch, issue activity, warp instructions."""
    path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(path) as f:
            e = json.load(f).get(config, {}).get(kernel)
    except Exception:
        return None
    if e is not None:
        e = dict(e)
        e["current"] = e.get("src_hash") == kernel_src_hash()
    return e


def stats_of(xs):
    xs = sorted(xs)
    return {"median": statistics.median(xs), "min": xs[0], "max": xs[-1], "mean": statistics.mean(xs)}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, dev):
        self.dev = dev
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits", "-lms", "100",
                 "-i", str(self.dev)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        self.out = ""
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.out, _ = self.proc.communicate(timeout=5)
            except Exception:
                self.proc.kill()
                self.out = ""

    def summary(self):
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in (self.out or "").strip().splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[1]))
                smax = float(parts[2])
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


def cpu_model():
    """The host CPU the oracle ran on (/proc/cpuinfo model name)."""
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def cpu_baseline(cfg_name, n, s, d, target_s):
    """The oracle (oracle/tc_oracle.c) as it stands, on this host's cores, over a
    bounded vertex-stride sample of the same graph (full graph when it fits)."""
    import oracle
    oracle.set_threads(len(os.sched_getaffinity(0)))
    t0 = time.perf_counter()
    g = oracle.Graph(n, s, d)
    t_build = time.perf_counter() - t0
    # probe with a 1/256 stride sample, then size the sample to ~target_s
    t0 = time.perf_counter()
    _, e_probe = g.count_range(0, n, 256)
    t_probe = max(time.perf_counter() - t0, 1e-4)
    est_full = t_probe * 256
    stride = 1 if est_full <= target_s else max(1, int(est_full / target_s + 0.999))
    t0 = time.perf_counter()
    T_s, e_s = g.count_range(0, n, stride)
    dt = time.perf_counter() - t0
    m_edges = g.m_edges
    single = None
    if cfg_name in ("c1", "c2"):
        # the same count on ONE host thread (C1 and C2 also single-threaded)
        ncores = oracle.threads()
        oracle.set_threads(1)
        t1 = time.perf_counter()
        T1, e1 = g.count_range(0, n, stride)
        d1 = time.perf_counter() - t1
        oracle.set_threads(ncores)
        single = {"value": e1 / d1, "unit": UNIT, "cores": 1, "seconds": d1, "triangles_in_sample": T1}
    g.close()
    sample = ("full graph" if stride == 1 else
              f"every {stride}-th vertex as the lowest triangle vertex ({e_s} of {m_edges} DAG edges)")
    out = {"value": e_s / dt, "unit": UNIT, "cores": oracle.threads(), "cpu_model": cpu_model(), "kind": "oracle",
           "sample": f"{cfg_name}: node iterator over {sample}; oracle build {t_build:.1f}s excluded",
           "seconds": dt, "triangles_in_sample": T_s, "full": stride == 1}
    if single:
        out["single_thread"] = single
    return out


L2_NOTE = "L2 flushed (256 MiB write) between timed steps, outside the events"


def workload_config(cfg, args, n, m_tuples, m_edges, p):
    """The workload keys, identical in both arms (ours and --impl reference)."""
    return {"workload": f"{cfg.name}: {cfg.desc}", "path": args.path, "n": n, "tuples": m_tuples,
            "m_edges": m_edges, "p": p, "cut_rule": args.cut_rule, "orient": args.orient,
            "l2": L2_NOTE}


def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    from gen.configs import CONFIGS
    import oracle
    # under torchrun OMP_NUM_THREADS=1: the one reference process uses every host core
    oracle.set_threads(len(os.sched_getaffinity(0)))
    cfg = CONFIGS[args.config]
    n, s, d = cfg.generate()
    g = oracle.Graph(n, s, d)
    m_edges = g.m_edges
    t0 = time.perf_counter()
    _, e_probe = g.count_range(0, n, 256)
    t_probe = max(time.perf_counter() - t0, 1e-4)
    per_step = max(1.0, 60.0 / max(args.steps + args.warmup, 1))   # whole run ~1 min
    stride = max(1, int(t_probe * 256 / per_step + 0.999))
    rates, times = [], []
    for k in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        _, e = g.count_range(k % stride, n, stride)
        dt = time.perf_counter() - t0
        if k >= args.warmup:
            times.append(dt)
            rates.append(e / dt)
    g.close()
    value = statistics.median(rates)
    p = max(1, min(args.p or cfg.p, n))
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": max(ws, args.gpus),
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * statistics.median(times),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u32",
        "data": "synthetic",
        "config": workload_config(cfg, args, n, int(s.size), m_edges, p),
        "run": {"device": "host CPU (the oracle, oracle/tc_oracle.c; no GPU used)", "sample_stride": stride,
                "step": f"node iterator over every {stride}-th vertex as the lowest triangle vertex "
                        "(rotating offset); value = median over steps of sampled DAG edges / step time"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": oracle.threads(), "cpu_model": cpu_model(),
                         "kind": "oracle",
                         "sample": f"each step: node iterator over every {stride}-th vertex (rotating offset)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


class Comm:
    """Process-group plumbing for N>1: NCCL, one rank per GPU (the production path:
    the 8-byte count allreduce runs on the GPU stream).  With --shared-gpu (flow
    tests on a 1-GPU box only) ranks share a GPU and talk gloo with host tensors."""

    def __init__(self, ws, local, shared_ok=False):
        import torch
        import torch.distributed as dist
        self.ws, self.dist, self.torch = ws, dist, torch
        ndev = torch.cuda.device_count()
        if ws > ndev and not shared_ok:
            raise SystemExit(f"bench.py: {ws} ranks but {ndev} CUDA device(s) visible "
                             "(one process per GPU; --shared-gpu only for flow tests)")
        self.dev = local % max(ndev, 1)
        torch.cuda.set_device(self.dev)
        self.backend = None
        if ws > 1:
            self.backend = "nccl" if ndev >= ws else "gloo"
            if self.backend == "nccl":
                dist.init_process_group("nccl", device_id=torch.device("cuda", self.dev))
            else:
                dist.init_process_group("gloo")

    def allreduce_(self, t, op="sum"):
        if self.ws <= 1:
            return t
        dop = self.dist.ReduceOp.SUM if op == "sum" else self.dist.ReduceOp.MAX
        if self.backend == "nccl":
            self.dist.all_reduce(t, op=dop)
            return t
        h = t.cpu()
        self.dist.all_reduce(h, op=dop)
        t.copy_(h)
        return t

    def barrier(self):
        if self.ws > 1:
            self.dist.barrier()

    def close(self):
        if self.ws > 1:
            self.dist.destroy_process_group()


def golden_triangles(config):
    """Oracle count written by tests/golden/make_golden.py (oracle-only script)."""
    path = os.path.join(ROOT, "tests", "golden", "triangles.json")
    try:
        return json.load(open(path)).get(config, {}).get("triangles")
    except Exception:
        return None


def roofline_of(cfg_name, kernels, ms_step, peak, peak_src, vertex, sm_clock_mhz, sms):
    """roofline of the dominant S10 kernel.

    achieved/frac: LOGICAL bytes (the R19 staged-list model) per launch
    / the kernel's live CUDA-event time -- the metric's "% of HBM roofline".  Hub
    lists are re-read from L2, so this is an effective bandwidth that can exceed 1.
    What actually limits the kernel comes from the committed ncu capture of this
    config (DRAM bytes, issue activity): `bound` is "hbm" when DRAM is the busier
    unit, "alu" when instruction issue is."""
    dom = max(kernels, key=lambda k: k["ms"])
    nc = ncu_entry(cfg_name, dom["kernel"]) if not vertex else None
    r = {"bound": "hbm", "achieved": dom["achieved"], "peak": peak, "unit": "GB/s", "frac": dom["frac"],
         "traffic": None, "achieved_kind": "logical_bytes (R19 staged-list model; L2-served re-reads count)",
         "frac_nominal_8tbs": dom["achieved"] / NOMINAL_HBM_GBS, "peak_source": peak_src,
         "kernel": dom["kernel"] + ("<VTX> (S10 + t(v) atomics)" if vertex else " (S10 intersections)"),
         "kernel_ms": dom["ms"], "kernel_share_of_step": dom["ms"] / ms_step if ms_step else None,
         "alg_bytes_per_launch": dom["alg_bytes"], "model": "staged-list bytes, SURVEY 8(d) / DESIGN R19",
         "kernels": kernels}
    if nc:
        dram = nc.get("dram_bytes_per_launch")
        r["traffic"] = dram
        r["ncu"] = {k: nc.get(k) for k in ("source", "src_hash", "current", "l2_hit_pct", "issue_active_pct",
                                           "warp_inst_per_launch", "top_stall", "kernel_ms_under_ncu")}
        # fractions from the capture itself (its DRAM bytes over its own kernel time, its
        # issue-active ratio), so they stay consistent even when the capture is of an
        # older build (ncu.current false); the live event time gives dram_gbs_live
        dfrac = ifrac = None
        ncu_ms = None
        try:
            v, unit = str(nc.get("kernel_ms_under_ncu") or "").split()
            ncu_ms = float(v) * {"ms": 1.0, "s": 1e3, "us": 1e-3}[unit]
        except Exception:
            ncu_ms = None
        if dram is not None and ncu_ms:
            dgbs = dram / (ncu_ms / 1e3) / 1e9
            dfrac = dgbs / peak
            r["dram_gbs"] = dgbs
            r["dram_frac"] = dfrac
            r["dram_frac_nominal_8tbs"] = dgbs / NOMINAL_HBM_GBS
            if dom["ms"] > 0:
                r["dram_gbs_live"] = dram / (dom["ms"] / 1e3) / 1e9
        try:
            ifrac = float(str(nc.get("issue_active_pct")).split()[0]) / 100.0
        except Exception:
            ifrac = None
        inst = nc.get("warp_inst_per_launch")
        if ifrac is not None:
            r["issue"] = {"active_frac": ifrac, "basis": "ncu smsp__issue_active (one warp instruction per "
                          "SMSP per cycle is the issue peak)"}
            if inst and ncu_ms and sm_clock_mhz:
                r["issue"]["warp_inst_per_launch"] = inst
                r["issue"]["inst_per_logical_elem"] = inst / max(1.0, dom["alg_bytes"] / 4.0)
        if dfrac is not None and ifrac is not None:
            r["bound"] = "hbm" if dfrac >= ifrac else "alu"
            top = nc.get("top_stall") or ""
            if max(dfrac, ifrac) < 0.6 and "long_scoreboard" in top:
                r["limiter"] = (f"memory latency (top stall {top}; issue active {ifrac:.2f}, "
                                f"DRAM {dfrac:.2f} of peak)")
            else:
                r["limiter"] = ("HBM bandwidth" if r["bound"] == "hbm" else "instruction issue") + \
                               f" (issue active {ifrac:.2f}, DRAM {dfrac:.2f} of peak)"
    return r


def run_ours(args):
    import torch

    from gen.configs import CONFIGS
    import paper_2209_04541_b200 as pg

    ws, rank, local = dist_env()
    if ws > 1 and args.gpus not in (1, ws):
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={ws}")
    comm = Comm(ws, local, args.shared_gpu)
    dev = comm.dev
    cfg = CONFIGS[args.config]
    p = args.p or cfg.p
    n, s, d = cfg.generate()
    m_tuples = int(s.size)

    if ws > 1 and args.balance == "measured":
        # S8 with rank 0's measured task times broadcast to all ranks (DESIGN R22; untimed)
        from paper_2209_04541_b200 import dist as pgd
        b = pgd.build_blocks_balanced(n, s, d, p=p, cut_rule=args.cut_rule, orient=args.orient, light_held=args.light_held)
    elif args.budget_gb > 0:
        b = pg.build_blocks(n, s, d, p=p, cut_rule=args.cut_rule, orient=args.orient, light_held=args.light_held, device=dev, rank=rank, world_size=ws,
                            residency=pg.RESIDENT_HOST, device_budget_bytes=int(args.budget_gb * (1 << 30)))
    else:
        b = pg.build_blocks(n, s, d, p=p, cut_rule=args.cut_rule, orient=args.orient, light_held=args.light_held, device=dev, rank=rank, world_size=ws)
    st0 = b.stats()
    m_edges = int(st0["m_edges"])
    # a real (non-legacy-default) stream: the library orders its work on it and the
    # CUDA events below are recorded on it
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    out = torch.zeros(1, dtype=torch.int64, device="cuda")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")   # > 126 MB L2
    vertex = args.path in ("vertex", "vertex2")
    tv_dev = torch.zeros(max(n, 1), dtype=torch.int64, device="cuda") if vertex else None
    b_rev = None
    if args.path == "vertex2":   # the reversed-order handle of the two-pass route (R24)
        b_rev = pg.build_blocks(n, s, d, p=p, cut_rule=args.cut_rule, orient=args.orient, light_held=args.light_held, device=dev, rank=rank, world_size=ws,
                                reverse_order=True)

    def step():
        if b_rev is not None:
            # t(v): lowest+middle roles on the forward handle, + lowest on the reversed one
            b.vertex_triangles(stream=stream, out=tv_dev, sync=False, roles="low+mid")
            b_rev.vertex_triangles(stream=stream, out=tv_dev, sync=False, roles="low", accumulate=True)
            comm.allreduce_(tv_dev)
            return
        if vertex:
            # per-vertex t(v) on the device, then one allreduce of the n-vector
            b.vertex_triangles(stream=stream, out=tv_dev, sync=False)
            comm.allreduce_(tv_dev)
            return
        b.triangle_count(stream=stream, d_count=out.data_ptr(), sync=False)
        comm.allreduce_(out)            # S11: one 8-byte allreduce of the per-rank counts

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    T = int(tv_dev.sum().item()) // 3 if vertex else int(out.item())

    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    kern_ms, light_ms, launches = [], [], 0
    with ClockSampler(dev) as clk:
        comm.barrier()
        torch.cuda.synchronize()
        for k in range(args.steps):
            flush.zero_()                       # L2 flush between timed steps (outside events)
            ev[k][0].record(stream)
            step()
            ev[k][1].record(stream)
            torch.cuda.synchronize()
            stk = b.stats()
            kern_ms.append(stk["ms_main_kernel_last"])
            light_ms.append(stk["ms_light_kernel_last"])
            launches += int(stk["launches_last"])
            if b_rev is not None:   # the second pass's kernels count toward the step too
                sr = b_rev.stats()
                kern_ms[-1] += sr["ms_main_kernel_last"]
                light_ms[-1] += sr["ms_light_kernel_last"]
                launches += int(sr["launches_last"])
        torch.cuda.synchronize()
        comm.barrier()
    step_ms = [a.elapsed_time(z) for a, z in ev]
    # every step's time is the max over ranks (the slowest rank ends the step); the
    # reported step time is the median over steps (median of runs)
    per_step = torch.tensor(step_ms, dtype=torch.float64, device="cuda")
    per_step_max = [float(x) for x in comm.allreduce_(per_step, "max").cpu()]
    per_rank = torch.zeros(ws, dtype=torch.float64, device="cuda")
    per_rank[rank] = statistics.median(step_ms)
    per_rank_ms = [float(x) for x in comm.allreduce_(per_rank).cpu()]
    sstat = stats_of(per_step_max)
    ms_per_step = sstat["median"]
    value = m_edges / (ms_per_step / 1e3)

    peak, peak_src = load_peaks()
    st = b.stats()
    alg = int(st["alg_bytes_local"])
    if vertex:
        # + the t(v) vector: zeroed and read once in rank space, written once in original ids
        alg += 3 * 8 * n
    if b_rev is not None:   # the reversed pass streams its own staged-model bytes
        alg += int(b_rev.stats()["alg_bytes_local"]) + 3 * 8 * n
    kms = statistics.median(kern_ms) if kern_ms else float("nan")
    lms = statistics.median(light_ms) if light_ms else 0.0
    alg_l = int(st["alg_bytes_light"]) + (int(b_rev.stats()["alg_bytes_light"]) if b_rev is not None else 0)

    def kern(name, ms, nbytes):
        ach = nbytes / (ms / 1e3) / 1e9 if ms > 0 else 0.0
        return {"kernel": name, "ms": ms, "alg_bytes": nbytes, "achieved": ach, "frac": ach / peak}
    # S10 runs as two kernels (DESIGN R20): warp-per-row k_tc_rows, thread-per-row k_tc_light
    kernels = [kern("k_tc_rows", kms - lms, alg - alg_l), kern("k_tc_light", lms, alg_l)]
    clocks = clk.summary()
    roofline = roofline_of(args.config, kernels, ms_per_step, peak, peak_src, vertex,
                           clocks.get("sm_mhz") or 1965.0, torch.cuda.get_device_properties(dev).multi_processor_count)
    roofline["s10_combined"] = kern("k_tc_rows + k_tc_light", kms, alg)
    roofline["items"] = {"heavy": int(st["items_heavy"]), "light": int(st["items_light"]),
                         "medium": int(st["items_medium"]), "light_held": int(st["light_held"]),
                         "ell_bytes": int(st["ell_bytes"])}

    # e2e: host-resident handle through the same public call, H2D inside the timed region
    e2e = None
    if not args.no_e2e and not vertex and args.budget_gb <= 0:
        bh = pg.build_blocks(n, s, d, p=p, cut_rule=args.cut_rule, orient=args.orient, light_held=args.light_held, device=dev, rank=rank, world_size=ws,
                             residency=pg.RESIDENT_HOST, host_permille=args.host_permille,
                             task_weights=getattr(b, "task_weights_used", None))
        for _ in range(max(1, args.warmup)):
            bh.triangle_count()
        comm.barrier()
        torch.cuda.synchronize()
        wall = []
        for _ in range(args.steps):
            flush.zero_()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            local_T = bh.triangle_count()      # H2D of blocks + count + D2H of the count
            tt = torch.tensor([local_T], dtype=torch.int64, device="cuda")
            comm.allreduce_(tt)
            tt.item()
            wall.append(time.perf_counter() - t0)
        e_t = torch.tensor(wall, dtype=torch.float64, device="cuda")
        e_s = statistics.median(float(x) for x in comm.allreduce_(e_t, "max").cpu())
        sh = bh.stats()
        e2e = {"value": m_edges / e_s, "unit": UNIT,
               "h2d_bytes_per_step": int(sh["h2d_bytes_last"]), "d2h_bytes_per_step": 8,
               "ms_per_step": 1e3 * e_s, "timer": "host wall clock around the public call, median of steps, "
                                                 "max over ranks"}
        if args.host_permille:   # NEXT-3: sparsest pieces counted by host threads (no H2D for them)
            e2e["host_permille"] = args.host_permille
            e2e["ms_host_share"] = float(sh["ms_host_last"])
        bh.free()

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu and not vertex:
        cpu = cpu_baseline(cfg.name, n, s, d, args.cpu_seconds)

    if rank == 0:
        line = {
            "metric": METRIC if not vertex else "per-vertex triangle-count edges/sec (|E|/time)",
            "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "weak" if ws > 1 else "strong", "vs_baseline": None, "dtype": "u32", "data": "synthetic",
            "config": workload_config(cfg, args, n, m_tuples, m_edges, int(st["p"])),
            "run": {"step_ms": sstat, "per_rank_ms": per_rank_ms, "triangles": T, "tasks": int(st["ntasks"]),
                    "wedges": int(st["wedges"]), "alg_bytes": int(st["alg_bytes_total"]),
                    "build_ms": float(st0["ms_build"]), "parallelism": f"task-parallel x{ws}",
                    "balance": args.balance if ws > 1 else None, "comm": comm.backend,
                    "residency": (f"host-streamed through a {args.budget_gb:g} GB device budget, "
                                  f"{int(st['waves'])} waves, H2D {int(st['h2d_bytes_last'])} B + D2D reuse "
                                  f"{int(st['d2d_bytes_last'])} B per count "
                                  "inside the timed region") if args.budget_gb > 0 else "device",
                    "timer": "CUDA events per step on the launch stream; per step the max over ranks; "
                             "value from the median step"},
            "roofline": roofline,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches,
            "clocks": clocks,
        }
        if vertex:
            line["vertex_route"] = ("two-pass (low+mid forward, low reversed; R24)" if b_rev is not None
                                    else "one-pass (all roles)")
        gold = golden_triangles(args.config)
        if cpu and cpu.get("full"):
            line["parity"] = {"oracle_triangles": cpu["triangles_in_sample"],
                              "match": cpu["triangles_in_sample"] == T, "source": "oracle run in this job"}
        elif gold is not None:
            line["parity"] = {"oracle_triangles": gold, "match": gold == T,
                              "source": "tests/golden/triangles.json (oracle-only script)"}
        print(json.dumps(line), flush=True)
    b.free()
    if b_rev is not None:
        b_rev.free()
    comm.close()
    return 0


def run_cc(args):
    """NEXT-4: SV connected components on the TC blocks, one GPU.
    value = |E| / device time of one whole HOOK/LINK loop (CUDA events inside the call)."""
    import torch

    from gen.configs import CONFIGS
    import oracle
    import paper_2209_04541_b200 as pg
    ws, rank, local = dist_env()
    if ws > 1:
        if rank == 0:
            print(json.dumps({"metric": "connected-components edges/sec (|E|/time)", "unavailable":
                              "connected components run on one GPU (world_size 1)"}), flush=True)
        return 0
    torch.cuda.set_device(0)
    cfg = CONFIGS[args.config]
    p = args.p or cfg.p
    n, s, d = cfg.generate()
    b = pg.build_blocks(n, s, d, p=p, cut_rule=args.cut_rule, orient=args.orient, light_held=args.light_held, device=0)
    st0 = b.stats()
    m_edges = int(st0["m_edges"])
    lab = torch.empty(max(n, 1), dtype=torch.int32, device="cuda")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for _ in range(args.warmup):
        _, ncomp, iters = b.connected_components(out=lab)
    ms = []
    with ClockSampler(0) as clk:
        for _ in range(args.steps):
            flush.zero_()
            torch.cuda.synchronize()
            _, ncomp, iters = b.connected_components(out=lab)
            ms.append(b.stats()["ms_cc_last"])
    ms_step = statistics.mean(ms)
    peak, peak_src = load_peaks()
    # per SV round: the hook pass reads every col id (4 B) and C of both ends (8 B) per
    # edge plus one rowptr pair per row; the link pass reads and writes C (8 B per vertex)
    alg = iters * (12 * m_edges + 8 * n) + 4 * n
    ach = alg / (ms_step / 1e3) / 1e9
    line = {"metric": "connected-components edges/sec (|E|/time)", "value": m_edges / (ms_step / 1e3),
            "unit": UNIT, "n_gpus": 1, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u32",
            "data": "synthetic",
            "config": {"workload": f"{cfg.name}: {cfg.desc}", "path": "cc", "n": n, "m_edges": m_edges,
                       "p": int(st0["p"]), "components": ncomp, "sv_rounds": iters,
                       "l2": "flushed (256 MiB write) between timed steps",
                       "timer": "CUDA events inside pgabb_connected_components (HOOK/LINK loop + labels)"},
            "roofline": {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak,
                         "traffic": None, "kernel": "k_cc_hook + k_cc_link (all SV rounds)",
                         "alg_bytes_per_launch": alg, "peak_source": peak_src,
                         "model": "per round 12 B/edge + 8 B/vertex (+4 B/vertex labels)"},
            "clocks": clk.summary(), "gpu_launches": 2 * iters + 3}
    if not args.no_cpu:
        import time as _t
        oracle.set_threads(len(os.sched_getaffinity(0)))
        g = oracle.Graph(n, s, d)
        t0 = _t.perf_counter()
        want, k = g.components()
        dt = _t.perf_counter() - t0
        g.close()
        import numpy as np
        got = lab[:n].cpu().numpy().astype(np.uint32)
        line["cpu_baseline"] = {"value": m_edges / dt, "unit": UNIT, "cores": 1, "kind": "oracle",
                                "sample": "full graph: sequential union-find (oracle_components)"}
        line["parity"] = {"oracle_components": k, "match": bool(k == ncomp and np.array_equal(got, want))}
    b.free()
    print(json.dumps(line), flush=True)
    return 0


def main():
    args = parse()
    if args.impl == "ours" and args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        self_launch(args)
    if args.impl == "reference":
        return run_reference(args)
    if args.path == "cc":
        return run_cc(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
