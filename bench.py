"""Benchmark: MinkUNet scans/sec on SemanticKITTI-shaped synthetic scans
(BASELINE.json metric).

    python bench.py [--gpus N --steps K --warmup W --impl {engine,reference}]
                    [--strong S] [--model centerpoint] [--layer-csv PATH]

One process per GPU (torchrun for N > 1).  Scans are independent, so every
rank runs its own batch of scans packed into one batched SparseTensor with a
shared boundary, with no data-path collective.  Default: weak scaling, B = 8
scans per GPU per step (config 5's per-GPU shard; 64 scans at N = 8).
``--strong S``: config 5 as a fixed batch of S scans (64) assigned to the
ranks by LPT on voxel count (strong scaling).

`value`    whole-job scans/s with inputs resident in HBM (device-timed with
           CUDA events, max over ranks), L2 flushed between timed steps.
`e2e`      the same through the public API with host buffers: pinned H2D of
           coords + features, SparseTensor construction (validated),
           model forward, D2H of the logits (each rank's final output to
           host memory: the path's only "gather"), every step.
`roofline` the dominant kernel (algorithmic bytes / its event time), from K
           more steps instrumented with per-layer CUDA events.
`cpu_baseline` the UNMODIFIED reference package (baseline/_ref) running the
           same MinkUNet graph, one process per host core (rank 0, N = 1); a
           step's bounded sample is one azimuth sector (1/16 of a scan's
           voxels, equal-count cuts) per worker, counted as that fraction of
           a scan (~28 s per whole scan per core otherwise).
`--impl reference` times that CPU path alone (the reference arm): W warm-up
           and K timed steps of the same samples.
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
    ap.add_argument("--cpu-steps", type=int, default=12,
                    help="steps of the in-line cpu_baseline (each: one 1/16-scan sector per core)")
    ap.add_argument("--strong", type=int, default=None,
                    help="strong scaling over a fixed batch of S scans (config 5: 64)")
    ap.add_argument("--layer-csv", default=None,
                    help="write the per-(layer, stage) CUDA-event table (layer,stage,metric,value)")
    ap.add_argument("--dataflow", choices=("staged", "fused", "auto"), default="auto")
    ap.add_argument("--strategy", default=None,
                    help="JSON v1 strategy file with per-layer fused-kernel launch shapes "
                         "(default: the committed B200 MinkUNet-1.0x file; 'none' = heuristics)")
    ap.add_argument("--clock-ms", type=int, default=5, help="clock sampling period (0: off)")
    ap.add_argument("--gather", choices=("host", "rank0"), default="host",
                    help="e2e output gather: host = each rank downloads its own scans' logits "
                         "(default); rank0 = NCCL gather of all logits to rank 0, then its D2H")
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


# ------------------------------------------------------------------ CPU path (the reference)

_W = {}


def _cpu_worker_init(width, model, scans):
    for k in ("OPENBLAS_NUM_THREADS", "OMP_NUM_THREADS", "MKL_NUM_THREADS", "NUMBA_NUM_THREADS"):
        os.environ[k] = "1"
    from oracle.reference_runner import import_reference, model_tables
    S = import_reference()
    _W.update(S=S, width=width, model=model, scans=scans)
    if model == "minkunet":  # numpy-only module: workers never import torch
        _W["params"] = model_tables("minkunet").build_params(width, 4, 0)
    else:
        _W["params"] = model_tables("centerpoint").build_params(5, 0)
    # numba JIT of the reference's movement kernels, outside any timed step
    rng = np.random.default_rng(0)
    keys = np.sort(rng.choice(16 ** 3, 600, replace=False))
    c = np.stack([np.zeros_like(keys), keys // 256, keys // 16 % 16, keys % 16], 1)
    t = S.quantize_features(S.SparseTensor(c, rng.standard_normal((600, 8)), 1, (16, 16, 16)),
                            S.PrecisionMode.FP16_STORAGE)
    S.sparse_conv_forward(t, S.WeightTensor(rng.standard_normal((27, 8, 8)), 3, 3),
                          S.LayerSpec(3, 1, 8, 8), options=S.ExecOptions(index_kind="hash"))


# The reference's CPU path needs ~28 s per whole MinkUNet-1.0x scan per core,
# so a step's sample is one azimuth sector per worker: each scan's voxels
# sorted by azimuth around the scan's centroid and cut into CPU_SECTORS runs of
# equal voxel count (balanced workers); throughput counts processed voxels as
# fractions of their scan.  Measured single-process, one thread: a 1/16 sector
# costs 29 s per scan-equivalent, a whole scan 28 s (1/48: 38 s, fixed per-layer
# overheads), so 1/16 sectors sample the whole-scan rate.
CPU_SECTORS = 16


def scan_sectors(scan, sectors=CPU_SECTORS):
    c, f, b = scan
    x, y = c[:, 1].astype(np.float64), c[:, 2].astype(np.float64)
    order = np.argsort(np.arctan2(y - y.mean(), x - x.mean()), kind="stable")
    return [(c[np.sort(part)], f[np.sort(part)], b, part.shape[0] / c.shape[0])
            for part in np.array_split(order, sectors)]


def _cpu_worker_run(i):
    """Item i: sector (i // scans) % CPU_SECTORS of scan i % scans.
    Returns (seconds, fraction of a scan processed)."""
    from oracle import reference_runner as R
    scans = _W["scans"]
    if "sectors" not in _W:
        _W["sectors"] = [scan_sectors(sc_) for sc_ in scans]
    c, f, b, frac = _W["sectors"][i % len(scans)][(i // len(scans)) % CPU_SECTORS]
    t0 = time.perf_counter()
    if _W["model"] == "minkunet":
        R.minkunet_reference(_W["S"], _W["params"], _W["width"], c, f, b)
    else:
        R.centerpoint_reference(_W["S"], _W["params"], c, f, b)
    return time.perf_counter() - t0, frac


class CpuPath:
    """The reference's own CPU implementation (the unmodified `sparseconv`
    package through its public API, oracle/reference_runner.py) on P worker
    processes, one host core each; a step = every worker runs one azimuth
    sector (1/CPU_SECTORS of a scan's voxels) of the workload's scans."""

    def __init__(self, width, scans, procs, model="minkunet"):
        import multiprocessing as mp
        self.procs = max(1, procs)
        # one thread per worker process: the BLAS / OpenMP / numba pools size
        # themselves when the child imports numpy, before any initializer runs,
        # so the limits go into the environment the children are spawned with
        # (measured: a sector took ~20 s in an oversubscribed pool, 0.55 s alone)
        keys = ("OPENBLAS_NUM_THREADS", "OMP_NUM_THREADS", "MKL_NUM_THREADS", "NUMBA_NUM_THREADS")
        saved = {k: os.environ.get(k) for k in keys}
        os.environ.update({k: "1" for k in keys})
        try:
            self.pool = mp.get_context("spawn").Pool(self.procs, _cpu_worker_init,
                                                     (width, model, scans))
        finally:
            for k, v in saved.items():
                if v is None:
                    os.environ.pop(k, None)
                else:
                    os.environ[k] = v
        self.cursor = 0

    def run(self, steps: int, timeout_s: float = 900.0):
        """``steps`` x P samples through the pool as one stream (a worker
        takes the next sample when it finishes one; no barrier between
        steps).  Returns (seconds, scans processed)."""
        items = list(range(self.cursor, self.cursor + steps * self.procs))
        self.cursor += len(items)
        t0 = time.perf_counter()
        # a bounded wait: a worker that died would otherwise hang the pool
        res = self.pool.map_async(_cpu_worker_run, items, chunksize=1).get(timeout_s)
        return time.perf_counter() - t0, float(sum(r[1] for r in res))

    def step(self, timeout_s: float = 600.0):
        return self.run(1, timeout_s)

    def close(self):
        self.pool.terminate()
        self.pool.join()


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_cores():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def run_cpu(args, scans, steps, warmup=0):
    """Scan sectors on every host core through the reference: ``warmup``
    then ``steps`` steps' worth of samples streamed through the pool.
    Returns (value, steps, secs, procs, scans done)."""
    procs = min(cpu_cores(), 64)
    cpu = CpuPath(args.width, scans, procs, args.model)
    try:
        if warmup:
            cpu.run(warmup)
        secs, done = cpu.run(steps)
    finally:
        cpu.close()
    return done / secs, steps, secs, cpu.procs, done


def run_reference(args):
    """--impl reference: rank 0 alone times the reference's CPU path; the
    other ranks exit without work."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    B = args.scans_per_gpu if args.strong is None else args.strong
    scans = load_scans(range(B), args.model)
    METRIC, UNIT = metric_unit(args)
    value, steps, secs, procs, done = run_cpu(args, scans, steps=args.steps,
                                              warmup=args.warmup)
    name = "MinkUNet" if args.model == "minkunet" else "CenterPoint-style encoder"
    sample = (f"{procs} single-threaded worker processes x 1 azimuth sector (1/{CPU_SECTORS} of a "
              f"scan's voxels) per step, streamed ({name} "
              f"{args.width if args.model == 'minkunet' else ''}, FP16 storage, hash index), "
              f"{steps} timed steps after {args.warmup} warm-up: {done:.2f} scans in {secs:.1f} s; "
              f"the unmodified reference package (baseline/_ref) through its own API")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": args.gpus, "steps": steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * secs / steps, "higher_is_better": True,
        "scaling": "weak" if args.strong is None else "strong",
        "vs_baseline": None, "dtype": "f16-storage/f32-accumulate", "data": DATA,
        "config": workload_config(args, args.gpus, scans),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": procs, "kind": "reference",
                         "sample": sample, "cpu": cpu_model()},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


DATA = "synthetic (raycast LiDAR scans, random-init weights)"
DEBUG_ALLOC = os.environ.get("SCB_BENCH_DEBUG_ALLOC") == "1"
# per-layer fused-kernel launch shapes tuned on a B200 for the MinkUNet-1.0x
# 8-scan workload (tools/tune_minkunet.py)
DEFAULT_STRATEGY = ROOT / "paper_2204_10319_b200" / "configs" / "minkunet_b200_shapes.json"


def workload_config(args, world, scans):
    """Identical for both arms (same data, same graph)."""
    vox = int(round(np.mean([sc_[0].shape[0] for sc_ in scans]))) if scans else 0
    if args.model == "centerpoint":
        work = (f"CenterPoint-style sparse encoder (21 k3 layers, 4 strided) on nuScenes-shaped "
                f"10-sweep clouds (~{vox // 1000}k voxels each, 0.075 m, 5 channels), FP16 storage")
        name = "CenterPoint-encoder"
    else:
        work = (f"MinkUNet {args.width}x on SemanticKITTI-shaped raycast scans "
                f"(~{vox // 1000}k voxels each, 0.05 m, 4 channels), FP16 storage")
        name = f"MinkUNet-{args.width}x"
    if args.strong is None:
        batch = {"global_batch": args.scans_per_gpu * world, "scans_per_gpu": args.scans_per_gpu,
                 "parallelism": f"scan-sharded x{world} (weak: {args.scans_per_gpu} scans per GPU)"}
    else:
        batch = {"global_batch": args.strong, "scans_per_gpu": None,
                 "parallelism": f"scan-sharded x{world} (strong: {args.strong} scans, LPT by "
                                f"voxel count)"}
    return dict({"workload": work, "model": name, "voxels_per_scan_mean": vox,
                 "l2": "flushed (256 MiB write) before every timed step; per-step buffers >> L2"},
                **batch)


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

def assign_scans(args, rank, world):
    """Seeds this rank runs: weak = its own block of B; strong = an LPT
    share (by voxel count) of the fixed S-scan batch."""
    from paper_2204_10319_b200.sharding import lpt_assign, shard_seeds
    if args.strong is None:
        return shard_seeds(rank, world, args.scans_per_gpu)
    sizes = [s[0].shape[0] for s in load_scans(range(args.strong), args.model)]
    return sorted(lpt_assign(sizes, world)[rank])


def layer_table_rows(samples, steps):
    """(layer, stage) -> ms per step, in the reference LatencyBreakdown's
    long format (reference bench.py:26-76: layer,stage,metric,value)."""
    rows = []
    for (layer, stage), secs in samples.items():
        rows.append((layer, stage, "ms", 1e3 * secs / steps))
    return rows


def main():
    args = parse()
    import faulthandler
    # a stuck run leaves its stacks in the log instead of only a timeout
    faulthandler.dump_traceback_later(900, exit=False)
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
    dev = torch.device("cuda", local)
    if world > 1:
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        dist.init_process_group("nccl", device_id=dev)
        probe = torch.ones(1, device=dev)
        dist.all_reduce(probe)  # communicator up before any timing
        print(f"[bench] rank {rank}: NCCL communicator size {dist.get_world_size()} "
              f"(all_reduce probe {int(probe.item())})", file=sys.stderr, flush=True)

    seeds = assign_scans(args, rank, world)
    scans = load_scans(seeds, args.model)
    B = len(scans)
    all_scans = scans if (world == 1 and args.strong is None) else \
        load_scans(range(args.strong if args.strong else args.scans_per_gpu), args.model)
    coords, feats, boundary = pack(scans)
    if args.model == "minkunet":
        strat = args.strategy
        if strat is None and args.width == 1.0 and DEFAULT_STRATEGY.exists():
            strat = str(DEFAULT_STRATEGY)
        if strat == "none":
            strat = None
        model = EngineMinkUNet(args.width, 4, 0, strategy=strat)
        args.strategy_used = Path(strat).name if strat else None
    else:
        model = EngineCenterPoint(5, 0)
    coords_d = torch.from_numpy(coords.astype(np.int32)).to(dev)
    feats_d = torch.from_numpy(feats).to(dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    # one large cached segment up front: later per-step allocations split it
    # instead of calling cudaMalloc inside a timed step
    # (and the small-block pool: blocks < 1 MiB come from 2 MiB segments of
    # their own; a new one inside a timed step measured a 50-135 ms host stall)
    def _reserve(big, small_blocks):
        r = torch.empty(big, dtype=torch.uint8, device=dev)
        smalls = [torch.empty(512 << 10, dtype=torch.uint8, device=dev)
                  for _ in range(small_blocks)]
        del r, smalls
    _reserve(16 << 30, 256)
    for side in (getattr(model, "map_stream", None), getattr(model, "chain_stream", None)):
        if side is not None:  # the mapping streams' own pools
            with torch.cuda.stream(side):
                _reserve(2 << 30, 128)

    coords_ev = torch.cuda.Event()
    coords_ev.record()
    pipe = {"next": None}

    def make_input():
        t = sc.SparseTensor(coords_d, feats_d, 1, boundary, B, validate=False)
        return sc.quantize_features(t, sc.PrecisionMode.FP16_STORAGE)

    def step(timer=None, traffic=None):
        """One forward.  Uninstrumented steps run as a serving loop: batch
        i+1's level-0 maps and coordinate pyramid are queued (model.prefetch)
        right after batch i's convolutions, on the mapping streams, so they
        run beside them; every step still builds all of its maps."""
        opts = sc.ExecOptions(timer=timer, traffic_log=traffic, index_kind="hash",
                              dataflow=args.dataflow)
        if timer is not None or traffic is not None or not hasattr(model, "prefetch"):
            pipe["next"] = None
            return model.forward(make_input(), opts)
        t = pipe["next"] if pipe["next"] is not None else make_input()
        out = model.forward(t, opts)
        pipe["next"] = make_input()
        model.prefetch(pipe["next"], opts, coords_ready=coords_ev)
        return out

    # algorithmic bytes per layer from one untimed pass;
    # the warm-up steps after it settle the allocator again
    traffic = []
    step(None, traffic)
    torch.cuda.synchronize()
    # W warm-up steps at least, and at least ~1.5 s of them: a fresh box
    # needs that long to settle clocks, lazy module loads and the allocator
    # (unsynchronised, like the timed loop: as many forwards in flight, so the
    # caching allocator's pools reach their steady-state size here)
    warm, w0 = 0, time.perf_counter()
    while warm < args.warmup or (time.perf_counter() - w0 < 1.5 and warm < 200):
        step()
        warm += 1
        if warm % 16 == 0:
            torch.cuda.synchronize()
    torch.cuda.synchronize()

    # ---------------- device-resident timed region (no instrumentation)
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
    t_start, t_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    # a rehearsal of the exact timed loop first (untimed): the caching
    # allocator's pools then already hold what K unsynchronised steps need,
    # so no cudaMalloc lands inside the timed steps
    for i in range(args.steps):
        flush.fill_(i & 0xFF)
        step()
    torch.cuda.synchronize()
    seg0 = torch.cuda.memory_stats(dev).get("segment.all.allocated", 0)
    switch0 = sys.getswitchinterval()
    sys.setswitchinterval(5e-4)  # let the clock-sampler thread in between host issues
    hw0 = time.perf_counter()
    t_start.record()
    for i in range(args.steps):
        flush.fill_(i & 0xFF)  # L2 flush ahead of the step's first input read
        evs[i][0].record()
        h0 = time.perf_counter()
        out = step()
        host_ms.append(round(1e3 * (time.perf_counter() - h0), 3))
        evs[i][1].record()
        if DEBUG_ALLOC:
            st = torch.cuda.memory_stats(dev)
            print(f"[alloc] step {i}: segments {st.get('segment.all.allocated', 0)} "
                  f"large {st.get('segment.large_pool.allocated', 0)} small "
                  f"{st.get('segment.small_pool.allocated', 0)} reserved "
                  f"{st.get('reserved_bytes.all.current', 0) >> 20} MiB", file=sys.stderr)
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
    step_ms = [round(a.elapsed_time(b), 4) for a, b in evs]
    total_s = torch.tensor(t_start.elapsed_time(t_end) / 1e3, device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(total_s, op=dist.ReduceOp.MAX)
    total_s = float(total_s)
    value = B * args.steps / total_s
    if world > 1:  # whole-job scans/s: every rank's scans over the max-over-ranks time
        nb = torch.tensor(float(B), device=dev, dtype=torch.float64)
        dist.all_reduce(nb)
        value = float(nb) * args.steps / total_s

    # ---------------- instrumented steps: per-(layer, stage) CUDA events
    timer = sc.StageTimer()
    torch.cuda.synchronize()
    for i in range(args.steps):
        flush.fill_(i & 0xFF)
        step(timer)
    torch.cuda.synchronize()
    samples = timer.samples
    roof, stage_summary = roofline(args, samples, traffic)
    if args.layer_csv and rank == 0:
        with open(args.layer_csv, "w") as fh:
            fh.write("layer,stage,metric,value\n")
            for r in layer_table_rows(samples, args.steps):
                fh.write(f"{r[0]},{r[1]},{r[2]},{r[3]:.6f}\n")

    # ---------------- end to end through the public API with host buffers
    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(args, sc, model, coords, feats, boundary, B, dev, world, UNIT, out)

    # ---------------- CPU baseline (rank 0, N = 1): the reference on whole scans
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        v, st, secs, procs, done = run_cpu(args, scans, steps=args.cpu_steps, warmup=2)
        cpu = {"value": v, "unit": UNIT, "cores": procs, "kind": "reference",
               "sample": f"{procs} single-threaded processes x 1 azimuth sector (1/{CPU_SECTORS} "
                         f"scan) per step, streamed, {st} steps after 2 warm-up: {done:.2f} scans "
                         f"in {secs:.1f} s: the unmodified reference package (baseline/_ref) "
                         f"through its own API on this workload's scans",
               "cpu": cpu_model()}

    if world > 1:
        dist.barrier()
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * total_s / args.steps,
            "ms_per_scan": 1e3 * total_s * world / (args.steps * max(1, B * world)),
            "higher_is_better": True, "scaling": "weak" if args.strong is None else "strong",
            "vs_baseline": None, "dtype": "f16-storage/f32-accumulate", "data": DATA,
            "config": workload_config(args, world, all_scans),
            "voxels_per_gpu_rank0": int(coords.shape[0]),
            "roofline": roof, "stages_ms_per_step": stage_summary, "cpu_baseline": cpu,
            "e2e": e2e, "gpu_launches": int(launches), "clocks": clk, "warmup_steps_run": warm,
            "step_ms": step_ms, "host_issue_ms": host_ms,
            "cuda_mallocs_in_timed_steps": seg_allocs,
            "kernel_shapes": getattr(args, "strategy_used", None) or "heuristic",
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def roofline(args, samples, traffic):
    """Roofline of the dominant kernel from the instrumented steps: its
    algorithmic bytes (index term 4 |M'|) or FLOPs per step
    over its summed CUDA-event time."""
    stages, mapping_levels = {}, {}
    for (layer, stage), s_ in samples.items():
        stages[stage] = stages.get(stage, 0.0) + s_
        if stage == "mapping":
            mapping_levels[layer] = mapping_levels.get(layer, 0.0) + s_
    K = args.steps
    bytes_by = {"gather": 0, "matmul": 0, "scatter": 0, "fused": 0}
    fused_dense_idx = 0
    flops = fused_flops = fused_exec = 0
    n_fused = n_gemm = 0
    for _, rec in traffic:
        bytes_by["gather"] += rec.get("gather_bytes", 0) * K
        bytes_by["matmul"] += rec.get("gemm_bytes", 0) * K
        bytes_by["scatter"] += rec.get("scatter_bytes", 0) * K
        bytes_by["fused"] += rec.get("fused_bytes", 0) * K
        fused_dense_idx += rec.get("fused_bytes_dense_index", 0) * K
        flops += rec.get("gemm_flops", 0) * K
        fused_flops += rec.get("fused_flops", 0) * K
        fused_exec += rec.get("fused_flops_executed", 0) * K
        n_fused += "fused_bytes" in rec
        n_gemm += "gemm_bytes" in rec
    peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) \
        if (ROOT / "MEASURED_PEAKS.json").exists() else {}
    hbm_peak = peaks.get("hbm_gbs", 6650.0)
    tc_peak = peaks.get("bf16_tflops_sustained", peaks.get("bf16_tflops", 1590.0))
    src = ("MEASURED_PEAKS.json (hbm_gbs; bf16_tflops_sustained: kernels timed inside a long step)"
           if peaks else "fallback 6.65 TB/s / 1.59 PFLOP/s (B200_PROFILING.md; "
                         "MEASURED_PEAKS.json absent)")
    dom = max(("gather", "matmul", "scatter", "fused"), key=lambda k: stages.get(k, 0.0))
    kernel_name = {"gather": "scb gather_kernel", "matmul": "scb grouped_gemm_f16_kernel (tcgen05)",
                   "scatter": "scb scatter_kernel",
                   "fused": "scb implicit_conv_f16_kernel + implicit_conv_pair_kernel (tcgen05 cta_group::1 / ::2, fused gather/GEMM/epilogue) + upconv_scatter_kernel (transposed k2 layers, scatter form)"}[dom]
    n_launch = max(1, n_fused if dom == "fused" else n_gemm)
    t_dom = max(stages.get(dom, 0.0), 1e-12)
    gbps = bytes_by[dom] / t_dom / 1e9
    measured = {}
    traffic_file = ROOT / "profiles" / "latest_traffic.json"
    if traffic_file.exists():
        measured = json.loads(traffic_file.read_text())
    if dom == "fused":
        tflops = fused_flops / t_dom / 1e12
        intensity = fused_flops / max(1, bytes_by[dom])
        tensor_bound = intensity > tc_peak * 1e12 / (hbm_peak * 1e9)
        roof = {"bound": "tensor" if tensor_bound else "hbm",
                "achieved": tflops if tensor_bound else gbps,
                "peak": tc_peak if tensor_bound else hbm_peak,
                "unit": "TFLOP/s" if tensor_bound else "GB/s"}
        roof["frac"] = roof["achieved"] / roof["peak"]
        roof["algorithmic_flops_per_launch"] = fused_flops / K / n_launch
        roof["arithmetic_intensity_flop_per_byte"] = intensity
        roof["hbm_frac"] = gbps / hbm_peak
        roof["hbm_frac_dense_index_bytes"] = fused_dense_idx / t_dom / 1e9 / hbm_peak
        roof["tensor_frac_useful"] = tflops / tc_peak
        roof["tensor_frac_executed"] = fused_exec / t_dom / 1e12 / tc_peak
    else:
        roof = {"bound": "hbm", "achieved": gbps, "peak": hbm_peak, "unit": "GB/s",
                "frac": gbps / hbm_peak}
    m = measured.get(dom, {})
    roof.update({
        "kernel": kernel_name,
        "kernel_ms_per_step": 1e3 * t_dom / K,
        "launches_per_step": n_launch,
        "traffic": m.get("dram_bytes_per_launch"),
        "traffic_note": (f"ncu dram read+write of one launch ({m.get('launch')}) vs its "
                         f"{m.get('algorithmic_bytes_per_launch')} algorithmic bytes; "
                         f"{measured.get('source')}") if m else None,
        "algorithmic_bytes_per_launch": bytes_by[dom] / K / n_launch,
        "peak_source": src,
        "timing": f"per-layer CUDA events on the compute stream over {K} instrumented steps "
                  f"(after the timed region, same workload)",
    })
    summary = {k: round(1e3 * v / K, 4) for k, v in sorted(stages.items())}
    summary["mapping_by_level"] = {k: round(1e3 * v / K, 4) for k, v in sorted(mapping_levels.items())}
    if stages.get("matmul"):
        roof["gemm_tflops"] = flops / stages["matmul"] / 1e12
    return roof, summary


def run_e2e(args, sc, model, coords, feats, boundary, B, dev, world, UNIT, out):
    """End to end through the public API with host buffers: per step the
    pinned H2D of coords + features, SparseTensor(validate="async"),
    quantize, model forward, D2H of the logits, on copy streams."""
    import collections
    import torch
    import torch.distributed as dist
    h_coords = torch.from_numpy(coords.astype(np.int32)).pin_memory()
    h_feats = torch.from_numpy(feats).pin_memory()
    rank = dist.get_rank() if world > 1 else 0
    to_rank0 = world > 1 and args.gather == "rank0"
    rows_per_rank = None
    if to_rank0:  # static per rank (same scans every step): exchanged once
        from paper_2204_10319_b200.sharding import gather_rows
        rows_per_rank = [None] * world
        dist.all_gather_object(rows_per_rank, int(out.features.shape[0]))
    out_rows = sum(rows_per_rank) if (to_rank0 and rank == 0) else \
        (0 if to_rank0 else int(out.features.shape[0]))
    h_out = torch.empty((max(out_rows, 1), out.features.shape[1]),
                        dtype=torch.float16).pin_memory()
    h2d_s, d2h_s = torch.cuda.Stream(), torch.cuda.Stream()
    NB = 4
    c_ring = [torch.empty(h_coords.shape, dtype=h_coords.dtype, device=dev) for _ in range(NB)]
    f_ring = [torch.empty(h_feats.shape, dtype=h_feats.dtype, device=dev) for _ in range(NB)]
    done = [None] * NB
    pending = collections.deque()
    counter = [0]

    opts_e = sc.ExecOptions(index_kind="hash", dataflow=args.dataflow)
    nxt = {"t": None, "k": None}

    def upload():
        """The next batch's pinned H2D (copy stream) and its SparseTensor."""
        k = counter[0] % NB
        counter[0] += 1
        cur = torch.cuda.current_stream()
        with torch.cuda.stream(h2d_s):
            if done[k] is not None:
                h2d_s.wait_event(done[k])
            c_ring[k].copy_(h_coords, non_blocking=True)
            f_ring[k].copy_(h_feats, non_blocking=True)
            # validation (its hash index is level 0's) on the copy stream, so
            # `up` covers everything the mapping streams read
            t = sc.SparseTensor(c_ring[k], f_ring[k], 1, boundary, B, validate="async")
            up = h2d_s.record_event()
        cur.wait_event(up)
        return k, sc.quantize_features(t, sc.PrecisionMode.FP16_STORAGE), up

    def e2e_step():
        """Serving loop: batch i's forward and download, then batch i+1's
        upload and its prefetched level-0 maps / coordinate pyramid (beside
        batch i's convolutions).  Every step moves one batch in and out."""
        cur = torch.cuda.current_stream()
        if nxt["t"] is None:
            k, t, _ = upload()
        else:
            k, t = nxt["k"], nxt["t"]
        o = model.forward(t, opts_e)
        res = o.features
        if to_rank0:  # the path's one data collective: NCCL gather to rank 0
            blocks = gather_rows(res, rows_per_rank, 0)
            res = torch.cat(blocks) if blocks is not None else None
        done[k] = cur.record_event()
        d2h_s.wait_event(done[k])
        with torch.cuda.stream(d2h_s):
            if res is not None:
                h_out[: res.shape[0]].copy_(res, non_blocking=True)
            pending.append((o, d2h_s.record_event()))
        while len(pending) > 3:
            pending.popleft()[1].synchronize()
        if hasattr(model, "prefetch"):
            nxt["k"], nxt["t"], up = upload()
            model.prefetch(nxt["t"], opts_e, coords_ready=up)
        return o

    warm_e, w0 = 0, time.perf_counter()
    while warm_e < args.warmup or (time.perf_counter() - w0 < 1.0 and warm_e < 200):
        e2e_step()
        warm_e += 1
        if warm_e % 16 == 0:
            torch.cuda.synchronize()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    gc.collect()
    gc.disable()
    for _ in range(args.steps):   # rehearsal of the timed loop (allocator pools)
        e2e_step()
    torch.cuda.current_stream().wait_stream(d2h_s)
    torch.cuda.synchronize()
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
    nb = torch.tensor(float(B), device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(es, op=dist.ReduceOp.MAX)
        dist.all_reduce(nb)
    return {"value": float(nb) * args.steps / float(es), "unit": UNIT,
            "h2d_bytes_per_step": int(h_coords.numel() * 4 + h_feats.numel() * 4),
            "d2h_bytes_per_step": int(out_rows * out.features.shape[1] * 2),
            "output_gather": ("NCCL gather of every rank's logits to rank 0, then rank 0's D2H"
                              if to_rank0 else "each rank's logits D2H to its own pinned host "
                              "buffer (no collective)"),
            "host_issue_ms": e_host, "warmup_steps_run": warm_e,
            "cuda_mallocs_in_timed_steps":
                torch.cuda.memory_stats(dev).get("segment.all.allocated", 0) - seg_e,
            "path": "pinned H2D (copy stream) -> SparseTensor(validate=async) -> quantize -> "
                    f"{args.model} forward -> D2H of the output features to this rank's pinned "
                    f"host buffer (copy stream)"}


if __name__ == "__main__":
    main()
