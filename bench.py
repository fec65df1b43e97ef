"""Benchmark: MinkUNet scans/sec on SemanticKITTI-shaped synthetic scans
(BASELINE.json metric).

    python bench.py [--gpus N --steps K --warmup W --impl {engine,reference}]

One process per GPU (torchrun for N > 1).  Scans are independent, so every
rank runs its own batch of scans (seeds rank*B .. rank*B+B-1, packed into one
batched SparseTensor with a shared boundary) with no data-path collective:
weak scaling.  Default workload = config 5's per-GPU shard: MinkUNet 1.0x,
FP16 feature storage, B = 8 scans per GPU per step (64 scans at N = 8).

`value`   whole-job scans/s with inputs resident in HBM (device-timed with
          CUDA events, max over ranks), L2 flushed between timed steps.
`e2e`     the same through the public API with host buffers: pinned H2D of
          coords + features, SparseTensor construction (validated),
          Network forward, D2H of the logits, every step.
`roofline` the dominant stage kernel (algorithmic bytes / its event time).
`cpu_baseline` the CPU oracle port of the same graph on this host (rank 0,
          N = 1), on a bounded sample (azimuth sectors of a scan).
`--impl reference` times that CPU path alone (the reference arm).
"""

from __future__ import annotations

import argparse
import gc
import json
import os
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

# (expandable_segments:True measured 50-500 ms host stalls on the second
# timed step: segment growth maps memory synchronously; not used)
if os.environ.get("SCB_EXPANDABLE") == "1":
    os.environ.setdefault("PYTORCH_CUDA_ALLOC_CONF", "expandable_segments:True")

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "MinkUNet scans/sec (SemanticKITTI shape)"
UNIT = "scans/s"
CP_METRIC = "CenterPoint-style encoder sweeps/sec (nuScenes shape, config 4)"
CP_UNIT = "sweeps/s"


def metric_unit(args):
    return (METRIC, UNIT) if args.model == "minkunet" else (CP_METRIC, CP_UNIT)
SECTORS = 8


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("engine", "reference"), default="engine")
    ap.add_argument("--width", type=float, default=1.0)
    ap.add_argument("--model", choices=("minkunet", "centerpoint"), default="minkunet",
                    help="minkunet: the BASELINE metric (configs 3/5); centerpoint: config 4")
    ap.add_argument("--scans-per-gpu", type=int, default=8)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--dataflow", choices=("staged", "fused", "auto"), default="auto")
    ap.add_argument("--clock-ms", type=int, default=5, help="clock sampling period (0: off)")
    return ap.parse_args()


# ------------------------------------------------------------------ data

CP_AZIMUTHS = 3000  # nuScenes-shaped sweeps of ~200k voxels


def load_scans(seeds, model="minkunet"):
    from paper_2204_10319_b200 import workloads
    cache = Path(os.environ.get("SCB_SCAN_CACHE", "/tmp/scb_scans"))
    out = []
    for s in seeds:
        f = cache / (f"scan{s}.npz" if model == "minkunet" else f"sweeps{s}_{CP_AZIMUTHS}.npz")
        if f.exists():
            d = np.load(f)
            out.append((d["c"], d["f"], tuple(int(x) for x in d["b"])))
            continue
        if model == "minkunet":
            c, fe, b = workloads.semantickitti_scan(s)
        else:
            c, fe, b = workloads.nuscenes_sweeps(s, azimuths=CP_AZIMUTHS)
        try:
            cache.mkdir(parents=True, exist_ok=True)
            np.savez(f, c=c, f=fe, b=np.array(b))
        except OSError:
            pass
        out.append((c, fe, b))
    return out


def pack(scans):
    """B scans -> one batched tensor with a shared boundary (SURVEY §8(e):
    bit-identical to separate runs)."""
    boundary = tuple(int(max(s[2][d] for s in scans)) for d in range(3))
    coords = np.concatenate([np.concatenate([np.full((s[0].shape[0], 1), i, np.int64),
                                             s[0][:, 1:]], 1) for i, s in enumerate(scans)])
    feats = np.concatenate([s[1] for s in scans]).astype(np.float32)
    return coords, feats, boundary


def sectors(scan, n=SECTORS):
    """Azimuth sectors of one scan (features hold absolute x, y)."""
    c, f, b = scan
    ang = np.mod(np.arctan2(f[:, 1], f[:, 0]), 2 * np.pi)
    sid = np.minimum((ang / (2 * np.pi / n)).astype(int), n - 1)
    return [(c[sid == k], f[sid == k], b) for k in range(n)]


# ------------------------------------------------------------------ CPU path (oracle port)

_W = {}


def _cpu_worker_init(width, model="minkunet"):
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    _W["width"], _W["model"] = width, model
    if model == "minkunet":
        from paper_2204_10319_b200.minkunet import build_params
        _W["params"] = build_params(width, 4, 0)
    else:
        from paper_2204_10319_b200.centerpoint import build_params
        _W["params"] = build_params(5, 0)


def _cpu_worker_run(item):
    from oracle import sparseconv_oracle as O
    c, f, b = item
    t0 = time.perf_counter()
    if _W["model"] == "minkunet":
        from paper_2204_10319_b200.minkunet import forward_oracle
        forward_oracle(_W["params"], _W["width"], c, O.quantize(f, "fp16"), b)
    else:
        from paper_2204_10319_b200.centerpoint import forward_oracle
        forward_oracle(_W["params"], c, O.quantize(f, "fp16"), b)
    return time.perf_counter() - t0


class CpuPath:
    """The reference's CPU path (oracle port) over P worker processes, each
    running the full MinkUNet graph on one azimuth sector (1/8 scan) per step."""

    def __init__(self, width, scans, procs, model="minkunet"):
        import multiprocessing as mp
        os.environ["OPENBLAS_NUM_THREADS"] = "1"
        os.environ["OMP_NUM_THREADS"] = "1"
        os.environ["MKL_NUM_THREADS"] = "1"
        self.items = [sec for s in scans for sec in sectors(s)]
        self.procs = max(1, min(procs, len(self.items)))
        self.pool = mp.get_context("spawn").Pool(self.procs, _cpu_worker_init, (width, model))
        self.cursor = 0

    def step(self):
        batch = [self.items[(self.cursor + i) % len(self.items)] for i in range(self.procs)]
        self.cursor += self.procs
        t0 = time.perf_counter()
        self.pool.map(_cpu_worker_run, batch, chunksize=1)
        return time.perf_counter() - t0, self.procs / SECTORS  # seconds, scans processed

    def close(self):
        self.pool.close()
        self.pool.join()


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def run_reference(args):
    """--impl reference: rank 0 alone times the CPU path; others exit."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    n_scans = 2
    scans = load_scans(range(n_scans), args.model)
    METRIC, UNIT = metric_unit(args)
    procs = min(os.cpu_count() or 1, 64)
    cpu = CpuPath(args.width, scans, procs, args.model)
    for _ in range(args.warmup):
        cpu.step()
    secs, done = 0.0, 0.0
    for _ in range(args.steps):
        s, d = cpu.step()
        secs += s
        done += d
    cpu.close()
    value = done / secs
    sample = (f"{cpu.procs} worker processes x 1 azimuth sector (1/{SECTORS} scan) of MinkUNet "
              f"{args.width}x per step, FP16 storage, oracle port (numpy/OpenBLAS 1 thread each)")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * secs / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f16-storage/f32-accumulate", "data": "synthetic",
        "config": workload_config(args, 1),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cpu.procs, "kind": "port",
                         "sample": sample, "cpu": cpu_model()},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def workload_config(args, world):
    if args.model == "centerpoint":
        work = (f"CenterPoint-style sparse encoder (21 k3 layers, 4 strided), "
                f"{args.scans_per_gpu} nuScenes-shaped 10-sweep clouds per GPU per step "
                f"(~200k voxels each, 0.075 m, 5 channels), FP16 storage")
        name = "CenterPoint-encoder"
    else:
        work = (f"MinkUNet {args.width}x, {args.scans_per_gpu} SemanticKITTI-shaped "
                f"raycast scans per GPU per step (~120k voxels each, 0.05 m), FP16 storage")
        name = f"MinkUNet-{args.width}x"
    return {"workload": work,
            "model": name, "global_batch": args.scans_per_gpu * world,
            "scans_per_gpu": args.scans_per_gpu, "parallelism": f"scan-sharded x{world}",
            "l2": "flushed (256 MiB write, on the mapping stream ahead of the step's input reads) "
                  "before every timed step; per-step buffers >> L2"}


# ------------------------------------------------------------------ clocks

class Clocks:
    """SM clock and throttle-reason samples during the timed region: an
    in-process NVML thread (sub-millisecond queries, so a ~100 ms region
    still gets tens of samples); nvidia-smi -lms as the fallback."""

    REASONS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20,
               "sw_power_cap": 0x4}

    def __init__(self, path):
        self.path = path
        self.proc = None
        self.thread = None
        self.samples = []
        self.window = None

    def start(self, period_ms=10, gpu_index=0):
        import threading
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(gpu_index)
            self.max_mhz = float(pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM))
        except Exception:  # no NVML: nvidia-smi
            return self._start_smi(max(period_ms, 20))
        self.stop_flag = False

        self.errors = 0

        def run():
            while not self.stop_flag:
                t = time.perf_counter()
                try:
                    mhz = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                except Exception:
                    self.errors += 1
                    time.sleep(period_ms / 1e3)
                    continue
                try:
                    rs = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                except Exception:
                    rs = 0
                    self.errors += 1
                self.samples.append((t, float(mhz), int(rs)))
                time.sleep(period_ms / 1e3)
        self.thread = threading.Thread(target=run, daemon=True)
        self.thread.start()

    def mark(self, t0, t1):
        """The timed region, in time.perf_counter() seconds."""
        self.window = (t0, t1)

    def _start_smi(self, period_ms):
        try:
            self.fh = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", "--query-gpu=index,clocks.sm,clocks.max.sm,power.draw,"
                 "clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
                 "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
                 "clocks_event_reasons.sw_power_cap", "--format=csv,noheader,nounits", "-lms", str(period_ms)],
                stdout=self.fh, stderr=subprocess.DEVNULL)
        except (OSError, FileNotFoundError):
            self.proc = None

    def stop(self, gpu_index):
        if self.thread is not None:
            self.stop_flag = True
            self.thread.join()
            lo, hi = self.window or (-1e30, 1e30)
            inside = [x for x in self.samples if lo <= x[0] <= hi]
            sel = inside or self.samples[-3:]
            reasons = sorted(n for n, bit in self.REASONS.items() if any(r & bit for _, _, r in sel))
            return {"sm_mhz": float(np.median([m for _, m, _ in sel])) if sel else None,
                    "sm_max_mhz": self.max_mhz, "reasons": reasons, "samples": len(inside),
                    "samples_total": len(self.samples), "nvml_errors": self.errors,
                    "source": "NVML thread, samples inside the timed region"}
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        self.proc.wait()
        self.fh.close()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            p = [x.strip() for x in line.split(",")]
            if len(p) < 9 or p[0] != str(gpu_index):
                continue
            try:
                sm.append(float(p[1]))
                mx = float(p[2])
            except ValueError:
                continue
            for name, v in zip(names, p[5:9]):
                if v.lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm), "source": "nvidia-smi -lms"}


# ------------------------------------------------------------------ engine

def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    import torch
    import torch.distributed as dist

    import paper_2204_10319_b200 as sc
    from paper_2204_10319_b200 import _native as nat
    from paper_2204_10319_b200.centerpoint import EngineCenterPoint
    from paper_2204_10319_b200.minkunet import EngineMinkUNet
    METRIC, UNIT = metric_unit(args)

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    B = args.scans_per_gpu

    from paper_2204_10319_b200.sharding import shard_seeds
    scans = load_scans(shard_seeds(rank, world, B), args.model)
    coords, feats, boundary = pack(scans)
    if args.model == "minkunet":
        model = EngineMinkUNet(args.width, 4, 0)
    else:
        model = EngineCenterPoint(5, 0)
    coords_d = torch.from_numpy(coords.astype(np.int32)).to(dev)
    feats_d = torch.from_numpy(feats).to(dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    # one large cached segment up front: later per-step allocations split it
    # instead of calling cudaMalloc inside a timed step
    reserve = torch.empty(16 << 30, dtype=torch.uint8, device=dev)
    del reserve

    ms = getattr(model, "mapping_stream", None) or torch.cuda.current_stream()

    def step(timer=None, traffic=None):
        # the batch's coordinate set lives on the mapping stream (maps of
        # batch i+1 overlap the convolutions of batch i)
        with torch.cuda.stream(ms):
            t = sc.SparseTensor(coords_d, feats_d, 1, boundary, B, validate=False)
        t = sc.quantize_features(t, sc.PrecisionMode.FP16_STORAGE)
        return model.forward(t, sc.ExecOptions(timer=timer, traffic_log=traffic,
                                               index_kind="hash", dataflow=args.dataflow))

    # algorithmic bytes per layer from one untimed pass (the
    # traffic log takes the host-planned path, the timed steps the sync-free
    # one); the warm-up steps after it settle the allocator again
    traffic = []
    step(None, traffic)
    torch.cuda.synchronize()
    # W warm-up steps at least, and at least ~1.5 s of them: a fresh box
    # needs that long to settle clocks, lazy module loads and the allocator
    warm, w0 = 0, time.perf_counter()
    while warm < args.warmup or (time.perf_counter() - w0 < 1.5 and warm < 200):
        step()
        torch.cuda.synchronize()
        warm += 1

    # ---------------- device-resident timed region
    timer = sc.StageTimer()
    clocks = Clocks(str(ROOT / f"gpurun_out/clocks_rank{rank}.csv")
                    if (ROOT / "gpurun_out").exists() else f"/tmp/clocks_rank{rank}.csv")
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    if args.clock_ms > 0:
        clocks.start(args.clock_ms, local)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    launches0 = nat.load().scb_launch_count()
    seg0 = torch.cuda.memory_stats(dev).get("segment.all.allocated", 0)
    host_ms = []
    gc.collect()
    gc.disable()  # no collector pauses inside the timed steps
    # One event pair brackets all K steps on the compute stream; the mapping
    # stream starts after it.  Each step begins with an L2 flush on the
    # mapping stream, ahead of that step's first read of its inputs, so the
    # flushes (and any mapping overlapping the previous step) are inside the
    # timed region.
    t_start, t_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    switch0 = sys.getswitchinterval()
    sys.setswitchinterval(5e-4)  # let the clock-sampler thread in between host issues
    hw0 = time.perf_counter()
    t_start.record()
    ms.wait_event(t_start)
    for i in range(args.steps):
        with torch.cuda.stream(ms):
            flush.fill_(i & 0xFF)
        evs[i][0].record()
        h0 = time.perf_counter()
        out = step(timer)
        host_ms.append(1e3 * (time.perf_counter() - h0))
        evs[i][1].record()
    t_end.record()
    torch.cuda.synchronize()
    clocks.mark(hw0, time.perf_counter())
    sys.setswitchinterval(switch0)
    if world > 1:
        dist.barrier()
    gc.enable()
    seg_allocs = torch.cuda.memory_stats(dev).get("segment.all.allocated", 0) - seg0
    launches = nat.load().scb_launch_count() - launches0
    clk = clocks.stop(local) if args.clock_ms > 0 else {"sm_mhz": None, "reasons": ["not sampled"]}
    step_ms = [a.elapsed_time(b) for a, b in evs]  # compute-stream span of each step
    total_s = torch.tensor(t_start.elapsed_time(t_end) / 1e3, device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(total_s, op=dist.ReduceOp.MAX)
    total_s = float(total_s)
    value = B * world * args.steps / total_s

    # ---------------- roofline of the dominant stage kernel
    stages = {}
    for (layer, stage), s in timer.samples.items():
        stages[stage] = stages.get(stage, 0.0) + s
    bytes_by = {"gather": 0, "matmul": 0, "scatter": 0, "fused": 0}
    flops = fused_flops = fused_exec = 0
    for _, rec in traffic * args.steps:  # one pass recorded, K timed
        bytes_by["gather"] += rec.get("gather_bytes", 0)
        bytes_by["matmul"] += rec.get("gemm_bytes", 0)
        bytes_by["scatter"] += rec.get("scatter_bytes", 0)
        bytes_by["fused"] += rec.get("fused_bytes", 0)
        flops += rec.get("gemm_flops", 0)
        fused_flops += rec.get("fused_flops", 0)
        fused_exec += rec.get("fused_flops_executed", 0)
    peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) \
        if (ROOT / "MEASURED_PEAKS.json").exists() else {}
    hbm_peak = peaks.get("hbm_gbs", 6650.0)
    tc_peak = peaks.get("bf16_tflops_sustained", peaks.get("bf16_tflops", 1590.0))
    src = ("MEASURED_PEAKS.json" if peaks
           else "of fallback 6.65 TB/s / 1.59 PFLOP/s (B200_PROFILING.md; MEASURED_PEAKS.json absent)")
    dom = max(("gather", "matmul", "scatter", "fused"), key=lambda k: stages.get(k, 0.0))
    kernel_name = {"gather": "scb gather_kernel", "matmul": "scb grouped_gemm_f16_kernel (tcgen05)",
                   "scatter": "scb scatter_kernel",
                   "fused": "scb implicit_conv_f16_kernel (tcgen05, fused gather/GEMM/scatter)"}[dom]
    n_launch = max(1, sum(1 for _, r in traffic if (("fused_bytes" in r) if dom == "fused"
                                                      else ("gemm_bytes" in r))))
    gbps = bytes_by[dom] / stages[dom] / 1e9
    measured = {}
    traffic_file = ROOT / "profiles" / "latest_traffic.json"
    if traffic_file.exists():
        measured = json.loads(traffic_file.read_text())
    if dom == "fused":
        # arithmetic intensity of the useful work decides the bound (ridge = peak ratio)
        tflops = fused_flops / stages[dom] / 1e12
        intensity = fused_flops / max(1, bytes_by[dom])
        tensor_bound = intensity > tc_peak * 1e12 / (hbm_peak * 1e9)
        roof = {"bound": "tensor" if tensor_bound else "hbm",
                "achieved": tflops if tensor_bound else gbps,
                "peak": tc_peak if tensor_bound else hbm_peak,
                "unit": "TFLOP/s" if tensor_bound else "GB/s"}
        roof["frac"] = roof["achieved"] / roof["peak"]
        roof["algorithmic_flops_per_launch"] = fused_flops / args.steps / n_launch
        roof["arithmetic_intensity_flop_per_byte"] = intensity
        roof["hbm_frac"] = gbps / hbm_peak
        roof["tensor_frac_useful"] = tflops / tc_peak
        roof["tensor_frac_executed"] = fused_exec / stages[dom] / 1e12 / tc_peak
    else:
        roof = {"bound": "hbm", "achieved": gbps, "peak": hbm_peak, "unit": "GB/s",
                "frac": gbps / hbm_peak}
    m = measured.get(dom, {})
    roof.update({
        "kernel": kernel_name,
        "traffic": m.get("dram_bytes_per_launch"),
        "traffic_note": (f"ncu dram read+write of one launch ({m.get('launch')}) vs its "
                         f"{m.get('algorithmic_bytes_per_launch')} algorithmic bytes; "
                         f"{measured.get('source')}") if m else None,
        "algorithmic_bytes_per_launch": bytes_by[dom] / args.steps / n_launch,
        "peak_source": src,
        "per_stage": {k: {"ms_per_step": 1e3 * stages.get(k, 0.0) / args.steps,
                          "GBps": (bytes_by[k] / stages[k] / 1e9) if stages.get(k) else None}
                      for k in ("gather", "matmul", "scatter", "fused")},
        "mapping_ms_per_step": 1e3 * stages.get("mapping", 0.0) / args.steps,
    })
    if stages.get("matmul"):
        roof["gemm_tflops"] = flops / stages["matmul"] / 1e12

    # ---------------- end to end through the public API with host buffers
    e2e = None
    if not args.no_e2e:
        h_coords = torch.from_numpy(coords.astype(np.int32)).pin_memory()
        h_feats = torch.from_numpy(feats).pin_memory()
        h_out = torch.empty(tuple(out.features.shape), dtype=torch.float16).pin_memory()

        # a serving loop: uploads and the output download on their own copy
        # streams, so batch i+1's H2D and batch i's D2H overlap compute.  Input
        # buffers are a ring reused once the batch that last used them is done
        # (no record_stream: its delayed block reuse cost cudaMallocs), and
        # each output is kept alive until its download finished.
        import collections
        h2d_s, d2h_s = torch.cuda.Stream(), torch.cuda.Stream()
        NB = 4
        c_ring = [torch.empty(h_coords.shape, dtype=h_coords.dtype, device=dev) for _ in range(NB)]
        f_ring = [torch.empty(h_feats.shape, dtype=h_feats.dtype, device=dev) for _ in range(NB)]
        done = [None] * NB
        pending = collections.deque()
        counter = [0]

        def e2e_step():
            k = counter[0] % NB
            counter[0] += 1
            cur = torch.cuda.current_stream()
            with torch.cuda.stream(h2d_s):
                if done[k] is not None:
                    h2d_s.wait_event(done[k])
                c_ring[k].copy_(h_coords, non_blocking=True)
                f_ring[k].copy_(h_feats, non_blocking=True)
            cur.wait_stream(h2d_s)
            # validated as a serving loop would: asynchronously, checked at the
            # forward's first host read (no stall on the previous batch)
            t = sc.SparseTensor(c_ring[k], f_ring[k], 1, boundary, B, validate="async")
            t = sc.quantize_features(t, sc.PrecisionMode.FP16_STORAGE)
            o = model.forward(t, sc.ExecOptions(index_kind="hash", dataflow=args.dataflow))
            done[k] = cur.record_event()
            d2h_s.wait_event(done[k])
            with torch.cuda.stream(d2h_s):
                h_out.copy_(o.features, non_blocking=True)
                pending.append((o, d2h_s.record_event()))
            while len(pending) > 3:
                pending.popleft()[1].synchronize()
            return o

        warm_e, w0 = 0, time.perf_counter()
        while warm_e < args.warmup or (time.perf_counter() - w0 < 1.0 and warm_e < 200):
            e2e_step()
            torch.cuda.synchronize()
            warm_e += 1
        if world > 1:
            dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        gc.collect()
        gc.disable()
        seg_e = torch.cuda.memory_stats(dev).get("segment.all.allocated", 0)
        e_host = []
        e0.record()
        for _ in range(args.steps):
            h0 = time.perf_counter()
            e2e_step()
            e_host.append(round(1e3 * (time.perf_counter() - h0), 2))
        torch.cuda.current_stream().wait_stream(d2h_s)  # the last download is inside the region
        e1.record()
        torch.cuda.synchronize()
        gc.enable()
        es = torch.tensor(e0.elapsed_time(e1) / 1e3, device=dev, dtype=torch.float64)
        if world > 1:
            dist.all_reduce(es, op=dist.ReduceOp.MAX)
        e2e = {"value": B * world * args.steps / float(es), "unit": UNIT,
               "h2d_bytes_per_step": int(h_coords.numel() * 4 + h_feats.numel() * 4),
               "host_issue_ms": e_host, "warmup_steps_run": warm_e,
               "cuda_mallocs_in_timed_steps":
                   torch.cuda.memory_stats(dev).get("segment.all.allocated", 0) - seg_e,
               "d2h_bytes_per_step": int(h_out.numel() * 2),
               "path": "pinned H2D (copy stream) -> SparseTensor(validate=async) -> quantize -> "
                       f"{args.model} forward -> D2H of the output features (copy stream)"}

    # ---------------- CPU baseline (rank 0, N = 1)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        procs = min(os.cpu_count() or 1, 64)
        path = CpuPath(args.width, scans[:2], procs, args.model)
        path.step()  # warm (spawn + imports)
        secs, done = 0.0, 0.0
        while secs < args.cpu_seconds:
            s, d = path.step()
            secs += s
            done += d
        path.close()
        cpu = {"value": done / secs, "unit": UNIT, "cores": path.procs, "kind": "port",
               "sample": f"{path.procs} processes x 1 azimuth sector (1/{SECTORS} scan) per round,"
                         f" {done:.2f} scans in {secs:.1f} s; oracle port of the same MinkUNet "
                         f"graph ({args.model}; numpy, 1 BLAS thread per process)",
               "cpu": cpu_model()}

    if world > 1:
        dist.barrier()
    if rank == 0:
        n_vox = int(coords.shape[0])
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * total_s / args.steps,
            "ms_per_scan": 1e3 * total_s / (args.steps * B), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f16-storage/f32-accumulate",
            "data": "synthetic (raycast LiDAR scans, random-init weights)",
            "config": dict(workload_config(args, world), voxels_per_gpu=n_vox),
            "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": int(launches),
            "clocks": clk, "warmup_steps_run": warm, "step_ms": step_ms, "host_issue_ms": host_ms,
            "cuda_mallocs_in_timed_steps": seg_allocs,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
