"""Benchmark: effective GFLOP/s (2mnk/t) of the memory-lean Winograd schedules on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C2] [--impl ours|reference]

Default workload (N=1): BASELINE config 2 -- C <- A*B + C over Z/65521Z with the
paper's 2-temporary accumulating schedule (acc2), m=k=n=4096, residues from
SplitMix64 seeds A=2, B=3, C=4 stored as float64, cutoff 256 (depth 4).
A step is one full multiplication with the inputs resident in HBM; the
400 MB of inputs exceed the 126 MB L2, so no flush is needed between steps.

Multi-GPU (one process per GPU; ``--gpus N`` re-executes itself under
torch.distributed.run when WORLD_SIZE is unset): the 7^L top-level Winograd
products of ONE multiplication are partitioned over the ranks
(paper_0707_2347_b200/dist.py: A and B broadcast over NCCL, operands formed on
the owning rank, products sent back and folded into C on the root), strong
scaling; ranks are timed on the device and the max over ranks is reported,
with every rank's peak extra bytes.

``--impl reference`` times the reference's own CPU implementation (the
unmodified winomem headers compiled into oracle/_ref) on the host cores.
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

METRIC = "effective GFLOP/s (2mnk/t) per schedule and peak extra HBM bytes, 1/2/4/8 B200"

CONFIGS = {
    "C1": dict(variant="std2", m=1024, k=1024, n=1024, cutoff=128, seed=1, alpha=1, beta=0,
               field="modp", desc="C<-AB mod 65521, std2 (2 temporaries), 1024^3, cutoff 128"),
    "C2": dict(variant="acc2", m=4096, k=4096, n=4096, cutoff=256, seed=2, alpha=1, beta=1,
               field="modp", desc="C<-AB+C mod 65521, acc2 (2 temporaries), 4096^3, cutoff 256"),
    "C3": dict(variant="iprect", m=8192, k=4096, n=8192, cutoff=256, seed=3, alpha=1, beta=0,
               field="modp",
               desc="C<-AB mod 65521, in-place rectangle (std2/ovl/ovr/ip on 4096^2 squares, "
                    "A and B clobbered), 8192x4096x8192, cutoff 256"),
    "C4": dict(variant="ipmm", m=16384, k=16384, n=16384, cutoff=512, seed=4, alpha=1, beta=0,
               field="modp", desc="C<-AB mod 65521, ipmm (read-only, first level classical), "
                                  "16384^3, cutoff 512"),
    "C5": dict(variant="std2", m=32768, k=32768, n=32768, cutoff=1024, seed=5, alpha=1, beta=0,
               field="real", desc="float64 C<-AB, std2, 32768^3, cutoff 1024"),
}


def peaks():
    try:
        d = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        return d.get("hbm_gbs", 6650.0), "measured (MEASURED_PEAKS.json)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


class Clocks:
    """SM clock / throttle sampler for the timed region (B200_PROFILING.md clocks
    line).  NVML is polled every millisecond from a thread, so even a few-ms
    timed region gets samples; nvidia-smi -lms 20 is the fallback."""

    NAMES = [("hw_slowdown", 0x8), ("hw_thermal_slowdown", 0x40),
             ("sw_thermal_slowdown", 0x20), ("sw_power_cap", 0x4)]

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []
        self.samples = []  # (sm_mhz, max_mhz, reason bits)
        self.stop = threading.Event()
        self.thread = None

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            mx = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
            get_reasons = getattr(pynvml, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
                pynvml.nvmlDeviceGetCurrentClocksThrottleReasons

            def poll():
                while not self.stop.is_set():
                    try:
                        self.samples.append((pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
                                             mx, int(get_reasons(h))))
                    except Exception:
                        pass
                    time.sleep(0.001)

            self.thread = threading.Thread(target=poll, daemon=True)
            self.thread.start()
            return self
        except Exception:
            self.thread = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index),
                 "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        self.stop.set()
        if self.thread:
            self.thread.join(timeout=1)
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        for (c, m, bits) in self.samples:
            sm.append(float(c))
            mx = float(m)
            for nm, bit in self.NAMES:
                if bits & bit:
                    reasons.add(nm)
        names = [nm for nm, _ in self.NAMES]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm),
                "source": "nvml 1 ms poll" if self.samples else "nvidia-smi -lms 20"}


def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def host_info():
    model = "unknown"
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"nproc": os.cpu_count(), "cpu_model": model}


def tensor_peaks():
    for rnd in ("r2", "r1"):
        f = os.path.join(ROOT, "profiles", rnd, "tensor_peaks.json")
        if os.path.exists(f):
            return json.load(open(f)), "measured (profiles/%s/tensor_peaks.json)" % rnd
    return {}, None


def relaunch_under_torchrun(args):
    """--gpus N > 1 outside torchrun: re-exec this command under
    torch.distributed.run with N ranks on this node (127.0.0.1 rendezvous)."""
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
           f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    os.execv(sys.executable, cmd)


# the reference's own single-threaded CPU path, one full multiplication per
# host thread; C4 at full size is ~30 min per thread and runs as its ipmm
# 4096^3 cutoff-128 proxy, marked same_config: false
REF_PROXY = {"C4": (4096, 128)}


def cpu_reference_rate(cfg, config, threads):
    """Run the reference run_variant (oracle/_ref, -O3 -DNDEBUG) on `threads`
    host threads at once, each on its own copy of the workload.  Returns
    (GFLOP/s aggregate, seconds, sample description, same_config)."""
    from concurrent.futures import ThreadPoolExecutor

    import numpy as np

    from oracle import oracle as O

    m, k, n, cutoff = cfg["m"], cfg["k"], cfg["n"], cfg["cutoff"]
    same = True
    if config in REF_PROXY:
        m = k = n = REF_PROXY[config][0]
        cutoff = REF_PROXY[config][1]
        same = False
    variant = cfg["variant"]
    # no reference schedule runs the in-place rectangle: its closest path is std2
    # on the same shape
    ref_variant = "std2" if variant == "iprect" else variant
    A = O.fill_random(m, k, cfg["seed"])
    B = O.fill_random(k, n, cfg["seed"] + 1)
    C0 = O.fill_random(m, n, cfg["seed"] + 2) if cfg["beta"] else np.zeros((m, n), np.uint32)

    def one(_):
        O.ref_run_variant(ref_variant, A, B, C0, cfg["alpha"], cfg["beta"], cutoff)

    t0 = time.perf_counter()
    with ThreadPoolExecutor(max_workers=threads) as ex:
        list(ex.map(one, range(threads)))
    dt = time.perf_counter() - t0
    sample = (f"{threads} concurrent reference run_variant('{ref_variant}') calls, each the full "
              f"{m}x{k}x{n} cutoff {cutoff} multiplication (oracle/_ref: the unmodified reference "
              f"headers at -O3 -DNDEBUG; the reference is single-threaded per multiply)")
    return threads * 2.0 * m * n * k / dt / 1e9, dt, sample, same


def run_reference_arm(args, cfg):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    from oracle import oracle as O
    if cfg["field"] == "real":
        print(json.dumps({"impl": "reference",
                          "unavailable": "no reference float64 path (SPEC.md:94)"}))
        return
    if not O.ref_available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref not built"}))
        return
    threads = os.cpu_count() or 1
    for _ in range(args.warmup):
        cpu_reference_rate(cfg, args.config, threads)
    rates, secs = [], []
    sample, same = "", True
    for _ in range(args.steps):
        r, dt, sample, same = cpu_reference_rate(cfg, args.config, threads)
        rates.append(r)
        secs.append(dt)
    value = statistics.median(rates)
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": value, "unit": "GFLOP/s",
        "n_gpus": max(world, args.gpus), "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * statistics.median(secs), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u32",
        "data": "synthetic (SplitMix64 seeds, residues mod 65521)",
        "config": {"workload": args.config + ": " + cfg["desc"], "variant": cfg["variant"],
                   "same_config": same},
        "cpu_baseline": {"value": value, "unit": "GFLOP/s", "cores": threads,
                         "kind": "reference", "sample": sample, "host": host_info()},
        "e2e": {"value": value, "unit": "GFLOP/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }))


def measure_rooflines(ctx, step, rep, real, config):
    """Replay the step with only one kernel class (measurement-only `subset`
    option) and report each class's algorithmic bytes (or limb ops) over its
    measured time.  The headline class is the one with the largest share of the
    step in the committed ncu launch list (scripts/ncu_launch_summary.py), else
    the longest replay; the frame GEMM's tensor fraction always rides along."""
    import torch

    stream = ctx.stream

    def subset_time(sub, reps=3):
        ctx.set_option("subset", sub)
        step()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        ctx.enter()
        e0.record(stream)
        for _ in range(reps):
            step()
        e1.record(stream)
        torch.cuda.synchronize()
        ctx.set_option("subset", 0)
        return e0.elapsed_time(e1) / 1e3 / reps

    t_add = subset_time(1)
    t_leaf = subset_time(2)
    t_frame = subset_time(3) if rep.fused_frames else 0.0
    parts = ({"prep": subset_time(4), "gemm": subset_time(5), "comb": subset_time(6)}
             if rep.fused_frames else {})
    hbm, hbm_src = peaks()
    tpk, tpk_src = tensor_peaks()
    rooflines = {
        "additions": {"bound": "hbm", "kernel": "k_group / k_addsub (block additions)",
                      "algorithmic_bytes_per_step": rep.add_bytes_issued, "seconds_per_step": t_add},
        "frame_prep": {"bound": "hbm", "kernel": "k_frame_prep_limbs (S/T + raw limb planes)",
                       "algorithmic_bytes_per_step": rep.frame_prep_bytes,
                       "seconds_per_step": parts.get("prep", 0.0)},
        "frame_gemm": {"bound": "tensor", "kernel": "k_gemm_direct (7 leaf products per launch, "
                                                    "tcgen05 kind::i8 on 2 x u8 limbs)",
                       "algorithmic_bytes_per_step": rep.frame_gemm_bytes,
                       "seconds_per_step": parts.get("gemm", 0.0),
                       "algorithmic_ops_per_step": 4 * rep.frame_leaf_flops},
        "frame_comb": {"bound": "hbm", "kernel": "k_frame_comb (U-chain, alpha/beta)",
                       "algorithmic_bytes_per_step": rep.frame_comb_bytes,
                       "seconds_per_step": parts.get("comb", 0.0)},
        "leaf_products": {"bound": "tensor",
                          "kernel": ("k_leaf_dmma (float64 DMMA leaves)" if real else
                                     "k_gemm_tma / k_gemm_i8 (unfused int8-limb leaves)"),
                          "algorithmic_bytes_per_step": None, "seconds_per_step": t_leaf,
                          "algorithmic_ops_per_step": (rep.leaf_flops - rep.frame_leaf_flops) *
                                                      (1 if real else 4)},
        "fused_frames": {"bound": "hbm",
                         "kernel": "fused leaf frames (prep + GEMM + comb, three launches)",
                         "algorithmic_bytes_per_step": rep.frame_bytes,
                         "seconds_per_step": t_frame},
    }
    for name, r_ in rooflines.items():
        b, t = r_["algorithmic_bytes_per_step"], r_["seconds_per_step"]
        if r_["bound"] == "tensor":
            # float64: 2mnk DMMA flops vs measured cuBLAS DGEMM; mod p: 4 x 2mnk
            # int8 limb ops vs measured cuBLASLt int8 (burst, clock-recorded)
            ops = r_["algorithmic_ops_per_step"]
            pk = tpk.get("fp64_tflops" if real else "int8_tops")
            if b and t:  # the operand / product plane stream it also moves
                r_["achieved_bytes_gbs"] = b / t / 1e9
            r_["achieved"] = ops / t / 1e12 if t and ops else None
            r_["peak"] = pk
            r_["unit"] = "TFLOP/s" if real else "TOP/s"
            r_["peak_source"] = tpk_src if pk else None
            r_["frac"] = r_["achieved"] / pk if r_["achieved"] and pk else None
            continue
        r_["achieved"] = b / t / 1e9 if b and t else None
        r_["peak"] = hbm
        r_["unit"] = "GB/s"
        r_["peak_source"] = hbm_src
        r_["frac"] = r_["achieved"] / hbm if r_["achieved"] else None
    single = [k_ for k_ in rooflines if k_ != "fused_frames" and rooflines[k_]["seconds_per_step"]]
    share, traffic_cls, basis = None, {}, "longest subset replay"
    for rnd in ("r2", "r1"):
        tfile = os.path.join(ROOT, "profiles", rnd, "ncu_launch_summary_%s.json" % config.lower())
        if os.path.exists(tfile):
            classes = json.load(open(tfile)).get("classes", {})
            share = {k_: v["share_of_step"] for k_, v in classes.items() if k_ in single}
            traffic_cls = classes
            basis = "largest share of the step in the ncu launch list (profiles/%s)" % rnd
            break
    if share:
        dominant = max(share, key=share.get)
    else:
        dominant = max(single, key=lambda k_: rooflines[k_]["seconds_per_step"])
    dom = rooflines[dominant]
    cls = traffic_cls.get(dominant)
    roof = {"bound": dom["bound"], "kernel": dom["kernel"], "achieved": dom["achieved"],
            "peak": dom["peak"], "unit": dom["unit"], "frac": dom["frac"],
            "traffic": cls.get("dram_bytes_per_step") if cls else None,
            "traffic_unit": "dram bytes per step (class total, ncu capture)",
            "peak_source": dom.get("peak_source"), "class": dominant, "class_basis": basis,
            "ncu_share_of_step": share,
            "algorithmic_bytes_per_step": dom["algorithmic_bytes_per_step"],
            "algorithmic_ops_per_step": dom.get("algorithmic_ops_per_step"),
            "kernel_seconds_per_step": dom["seconds_per_step"]}
    g = rooflines["frame_gemm"] if rep.fused_frames else rooflines["leaf_products"]
    roof["tensor_class"] = {k_: g.get(k_) for k_ in ("kernel", "achieved", "peak", "unit", "frac",
                                                     "peak_source", "seconds_per_step")}
    return rooflines, roof, {"additions": t_add, "leaf_products": t_leaf,
                             "fused_frames": t_frame}, parts


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C2", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--leaf", type=int, default=int(os.environ.get("WM_LEAF", 2)),
                    help="0 DMMA float64, 1 tcgen05 int8 limbs, 2 auto")
    ap.add_argument("--fuse", type=int, default=int(os.environ.get("WM_FUSE", 1)))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    args = ap.parse_args()
    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        run_reference_arm(args, cfg)
        return
    rank, world, local = dist_env()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        relaunch_under_torchrun(args)
    if world != args.gpus:
        sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    if os.environ.get("WM_BENCH_RANKS_ONLY"):  # launcher check (tests/test_bench_cli.py)
        print(json.dumps({"rank": rank, "world": world, "local_rank": local}), flush=True)
        return

    import numpy as np
    import torch

    import paper_0707_2347_b200 as W

    torch.cuda.set_device(local)
    # WM_BENCH_PARTITION=1: the partitioned path at N = 1 too (a one-rank NCCL
    # communicator), so the multi-GPU code path is exercised on one GPU
    if world > 1 or os.environ.get("WM_BENCH_PARTITION") == "1":
        import socket
        import torch.distributed as dist
        # communicator size in the log -- on stderr: stdout carries only the JSON line
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
        if "MASTER_PORT" not in os.environ:
            sk = socket.socket()
            sk.bind(("127.0.0.1", 0))
            os.environ["MASTER_PORT"] = str(sk.getsockname()[1])
            sk.close()
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", rank=rank, world_size=world,
                                device_id=torch.device("cuda", local))
        run_partitioned(args, cfg, rank, world, local)
        dist.destroy_process_group()
        return
    real = cfg["field"] == "real"
    m, k, n = cfg["m"], cfg["k"], cfg["n"]
    A = W.Matrix(m, k, device=local, real=real)
    B = W.Matrix(k, n, device=local, real=real)
    C = W.Matrix(m, n, device=local, real=real)
    ctx = A.ctx()
    ctx.set_option("leaf_kernel", args.leaf)
    ctx.set_option("fuse_frames", args.fuse)
    ctx.set_option("graphs", 1)
    for kv in filter(None, os.environ.get("WM_OPTS", "").split(",")):  # measurement sweeps
        opt_name, opt_val = kv.split("=")
        ctx.set_option(opt_name.strip(), int(opt_val))

    def reset_inputs():
        A.fill_random(cfg["seed"])
        B.fill_random(cfg["seed"] + 1)
        if cfg["beta"]:
            C.fill_random(cfg["seed"] + 2)
        else:
            C.fill_zero()

    def step():
        return W.run_variant(cfg["variant"], A, B, C, alpha=cfg["alpha"], beta=cfg["beta"],
                             cutoff=cfg["cutoff"])

    # parity of the very first multiplication against the golden hash
    reset_inputs()
    rep = step()
    torch.cuda.synchronize()
    if not real:
        gold = json.load(open(os.path.join(ROOT, "tests", "golden", "config_hashes.json")))
        h = "%016x" % C.hash()
        want = gold.get(args.config, {}).get("appendix_a")
        parity = {"c_hash": h, "golden": want, "ok": h == want}
    else:
        parity = real_parity(A, B, C, m, k, n, cfg)

    in_place = cfg["variant"] in ("iprect",)
    for _ in range(args.warmup):
        if in_place:
            reset_inputs()
        step()
    torch.cuda.synchronize()
    stream = ctx.stream
    small = 8 * (m * k + k * n + m * n) <= 126e6
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=f"cuda:{local}") \
        if small else None
    evs = []
    with Clocks(local) as clk:
        for _ in range(args.steps):
            if in_place:
                reset_inputs()  # A and B are clobbered: regenerate outside the timed events
            if flush is not None:
                flush.zero_()  # 256 MB write evicts L2 between timed steps
            ctx.enter()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            step()
            e1.record(stream)
            evs.append((e0, e1))
        torch.cuda.synchronize()
    times = [a.elapsed_time(b) / 1e3 for a, b in evs]
    t_step = sum(times) / len(times)
    flops = 2.0 * m * n * k
    value = flops / t_step / 1e9

    rooflines, roof, comps, frame_parts = measure_rooflines(ctx, step, rep, real, args.config)
    out = {
        "metric": METRIC, "value": value, "unit": "GFLOP/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_step * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic: SplitMix64 seeds A=%d B=%d C=%d, %s stored as float64" % (
            cfg["seed"], cfg["seed"] + 1, cfg["seed"] + 2,
            "uniform[-1,1)" if real else "residues mod 65521"),
        "config": {"workload": args.config + ": " + cfg["desc"], "variant": cfg["variant"],
                   "m": m, "k": k, "n": n, "cutoff": cfg["cutoff"], "alpha": cfg["alpha"],
                   "beta": cfg["beta"], "parallelism": "single",
                   "l2": "inputs (%.0f MB) %s L2; %s" % (
                       8 * (m * k + k * n + m * n) / 1e6,
                       ">" if 8 * (m * k + k * n + m * n) > 126e6 else "<=",
                       "no flush needed" if 8 * (m * k + k * n + m * n) > 126e6 else
                       "flushed between steps"),
                   "leaf_kernel": args.leaf, "fused_frames": bool(args.fuse)},
        "peak_extra_bytes": rep.peak_extra_bytes,
        "peak_extra_words": rep.peak_extra_words,
        "expected_peak_extra_words": W.expected_costs(cfg["variant"], m, k, n,
                                                      cfg["cutoff"]).peak_extra_words,
        "parity": parity,
        "breakdown_s": comps,
        "frame_breakdown_s": frame_parts,
        "rooflines": rooflines,
        "roofline": roof,
        "gpu_launches": rep.n_launches * args.steps,
        "launches_per_step": rep.n_launches,
        "clocks": clk.summary(),
    }
    if not args.no_e2e and not real:
        out["e2e"] = e2e(W, cfg, args, np, torch)
    if not args.no_cpu_baseline and not real:
        try:
            r, dt, sample, same = cpu_reference_rate(cfg, args.config, 1)
            out["cpu_baseline"] = {"value": r, "unit": "GFLOP/s", "cores": 1,
                                   "kind": "reference", "sample": sample, "same_config": same,
                                   "seconds": dt, "host": host_info()}
        except Exception as e:  # pragma: no cover
            out["cpu_baseline"] = {"value": None, "error": str(e)}
    print(json.dumps(out))


def real_parity(A, B, C, m, k, n, cfg):
    """float64: ||C - AB||_F / ||AB||_F estimated with Gaussian probe
    vectors (E ||dC x||^2 = ||dC||_F^2), the classical product applied as A (B x)
    in float64; stated tolerance 1e-12 * 2^depth."""
    import torch
    g = torch.Generator(device=C.t.device).manual_seed(1234)
    num = den = 0.0
    for _ in range(4):
        x = torch.randn(n, 1, dtype=torch.float64, device=C.t.device, generator=g)
        ref = A.t @ (B.t @ x)
        num += float(((C.t @ x) - ref).square().sum())
        den += float(ref.square().sum())
    depth = 0
    while (max(m, k, n) >> depth) > cfg["cutoff"]:
        depth += 1
    err = (num / den) ** 0.5
    return {"rel_frobenius_estimate": err, "probes": 4, "depth": depth,
            "tolerance": 1e-12 * 2 ** depth, "ok": err <= 1e-12 * 2 ** depth}


def run_partitioned(args, cfg, rank, world, local):
    """N > 1: the 7^L top-level Winograd products of ONE multiplication are
    spread over the ranks (paper_0707_2347_b200/dist.py: A and B broadcast,
    operands formed on the owning rank, products sent back and folded into C on
    the root); strong scaling, device-timed, max over ranks."""
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_0707_2347_b200 as W
    from paper_0707_2347_b200.dist import (CudaBackend, choose_levels, local_variant,
                                           makespan_bound, partitioned_multiply)

    real = cfg["field"] == "real"
    m, k, n = cfg["m"], cfg["k"], cfg["n"]
    levels = choose_levels(world, min(m, k, n), cfg["cutoff"])
    f = 2 ** levels
    lv = local_variant(cfg["variant"], m // f, k // f, n // f)
    be = CudaBackend(65521, lv, cfg["cutoff"], local, real=real)
    A = B = C = None
    if rank == 0:
        Am, Bm, Cm = (W.Matrix(m, k, device=local, real=real), W.Matrix(k, n, device=local, real=real),
                      W.Matrix(m, n, device=local, real=real))

        def reset():
            Am.fill_random(cfg["seed"])
            Bm.fill_random(cfg["seed"] + 1)
            if cfg["beta"]:
                Cm.fill_random(cfg["seed"] + 2)
            else:
                Cm.fill_zero()
        reset()
        A, B, C = Am.t, Bm.t, Cm.t

    def step():
        return partitioned_multiply(A, B, C, cfg["alpha"], cfg["beta"], be, levels=levels)

    parity = None
    st = step()
    torch.cuda.synchronize()
    if rank == 0:
        if real:
            parity = real_parity(Am, Bm, Cm, m, k, n, cfg)
        else:
            gold = json.load(open(os.path.join(ROOT, "tests", "golden", "config_hashes.json")))
            h = "%016x" % Cm.hash()
            want = gold.get(args.config, {}).get("appendix_a")
            parity = {"c_hash": h, "golden": want, "ok": h == want}
        reset()
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    dist.barrier()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    launches0 = be.launches
    with Clocks(local) as clk:
        e0.record()
        for _ in range(args.steps):
            st = step()
        e1.record()
        torch.cuda.synchronize()
    timed_launches = be.launches - launches0
    dist.barrier()
    t = torch.tensor([e0.elapsed_time(e1) / 1e3 / args.steps], device=f"cuda:{local}")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    t_step = float(t.item())

    # end to end: pinned host buffers in, C out, on the root, every step
    e2e_t = None
    h2d = 8 * (m * k + k * n + (m * n if cfg["beta"] else 0))
    if rank == 0:
        hA = A.to("cpu").pin_memory()
        hB = B.to("cpu").pin_memory()
        hC = C.to("cpu").pin_memory()
    dist.barrier()
    ts = []
    for _ in range(max(2, min(args.steps, 5))):
        torch.cuda.synchronize()
        dist.barrier()
        t0 = time.perf_counter()
        if rank == 0:
            A.copy_(hA, non_blocking=True)
            B.copy_(hB, non_blocking=True)
            if cfg["beta"]:
                C.copy_(hC, non_blocking=True)
        step()
        if rank == 0:
            hC.copy_(C, non_blocking=True)
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    tt = torch.tensor([statistics.median(ts)], device=f"cuda:{local}")
    dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    e2e_t = float(tt.item())

    per_rank = [None] * world
    dist.all_gather_object(per_rank, {"rank": rank, "products": len(st.products),
                                      "peak_extra_bytes": st.peak_extra_bytes,
                                      "bytes_sent": st.bytes_sent,
                                      "bytes_received": st.bytes_received,
                                      "timed_launches": timed_launches})
    out = None
    if rank == 0:
        # roofline of the per-rank work: one local product replayed by kernel class
        X = W.Matrix(m // f, k // f, device=local, real=real)
        Y = W.Matrix(k // f, n // f, device=local, real=real)
        P = W.Matrix(m // f, n // f, device=local, real=real)
        X.fill_random(11)
        Y.fill_random(12)
        ctx = X.ctx()

        def local_step():
            return W.run_variant(lv, X, Y, P, alpha=1, beta=0, cutoff=cfg["cutoff"])
        rep = local_step()
        rooflines, roof, comps, parts = measure_rooflines(ctx, local_step, rep, real,
                                                          args.config + "_local")
        out = {
            "metric": METRIC, "value": 2.0 * m * n * k / t_step / 1e9, "unit": "GFLOP/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": t_step * 1e3, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64",
            "data": "synthetic: SplitMix64 seeds A=%d B=%d C=%d" % (cfg["seed"], cfg["seed"] + 1,
                                                                   cfg["seed"] + 2),
            "config": {"workload": args.config + ": " + cfg["desc"], "variant": cfg["variant"],
                       "m": m, "k": k, "n": n, "cutoff": cfg["cutoff"],
                       "parallelism": f"{7 ** levels}-way product partition ({levels} Winograd "
                                      f"level(s)) over {world} GPUs: A/B broadcast, operands "
                                      f"formed per rank, P_t sent to the root (NCCL); local "
                                      f"schedule {lv}",
                       "makespan_bound": makespan_bound(world, 7 ** levels)},
            "parity": parity, "clocks": clk.summary(),
            "per_rank": per_rank,
            "peak_extra_bytes_max_rank": max(r["peak_extra_bytes"] for r in per_rank),
            "roofline": roof, "rooflines": rooflines,
            "gpu_launches": sum(r["timed_launches"] for r in per_rank),
            "e2e": {"value": 2.0 * m * n * k / e2e_t / 1e9, "unit": "GFLOP/s",
                    "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": 8 * m * n,
                    "seconds_per_step": e2e_t,
                    "timing": "host wall clock, pinned float64 buffers on the root, max over ranks"},
        }
        print(json.dumps(out))


def e2e(W, cfg, args, np, torch):
    """Same metric through the public host API: pinned u32 host buffers in,
    result out, host<->device copies inside the timed region."""
    m, k, n = cfg["m"], cfg["k"], cfg["n"]

    def host_input(rows, cols, seed):  # the package's own SplitMix64 fill, downloaded once (untimed)
        M = W.Matrix(rows, cols)
        M.fill_random(seed)
        out = M.to_u32()
        del M
        return out

    A = torch.from_numpy(host_input(m, k, cfg["seed"])).pin_memory().numpy()
    B = torch.from_numpy(host_input(k, n, cfg["seed"] + 1)).pin_memory().numpy()
    C0 = host_input(m, n, cfg["seed"] + 2) if cfg["beta"] else np.zeros((m, n), np.uint32)
    Cp = torch.from_numpy(C0.copy()).pin_memory().numpy()
    ctx = W.Context.get()
    ctx.set_option("leaf_kernel", args.leaf)
    ctx.set_option("fuse_frames", args.fuse)
    steps = max(3, min(args.steps, 5))
    for _ in range(2):
        Cp[...] = C0
        W.run_variant_host(cfg["variant"], A, B, Cp, cfg["alpha"], cfg["beta"], cfg["cutoff"])
    ts = []
    for _ in range(steps):
        Cp[...] = C0
        t0 = time.perf_counter()
        W.run_variant_host(cfg["variant"], A, B, Cp, cfg["alpha"], cfg["beta"], cfg["cutoff"])
        ts.append(time.perf_counter() - t0)
    t = statistics.median(ts)
    h2d = 4 * (m * k + k * n + (m * n if cfg["beta"] else 0))
    d2h = 4 * m * n
    if cfg["variant"] in ("iprect", "ipovmm"):
        d2h += 4 * (m * k + k * n)
    return {"value": 2.0 * m * n * k / t / 1e9, "unit": "GFLOP/s", "h2d_bytes_per_step": h2d,
            "d2h_bytes_per_step": d2h, "seconds_per_step": t,
            "timing": "host wall clock around the synchronous C-ABI call"}


if __name__ == "__main__":
    main()
