"""Tune the fused kernel's launch shape of every MinkUNet layer on the
bench's own workload (8 packed SemanticKITTI-shaped scans, MinkUNet 1.0x,
FP16) and write the JSON v1 strategy file bench.py loads by default.
Run on a B200:  python tools/tune_minkunet.py [out.json]"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2204_10319_b200 as sc  # noqa: E402
from paper_2204_10319_b200.autotune import save_strategy  # noqa: E402
from paper_2204_10319_b200.minkunet import EngineMinkUNet  # noqa: E402
from bench import DEFAULT_STRATEGY, load_scans, pack  # noqa: E402


def main():
    out = sys.argv[1] if len(sys.argv) > 1 else str(DEFAULT_STRATEGY)
    c, f, b = pack(load_scans(range(8)))
    model = EngineMinkUNet(1.0, 4, 0)
    t = sc.quantize_features(sc.SparseTensor(torch.from_numpy(c.astype(np.int32)).cuda(),
                                             torch.from_numpy(f).cuda(), 1, b, 8),
                             sc.PrecisionMode.FP16_STORAGE)
    opts = sc.ExecOptions(dataflow="auto")
    model.forward(t, opts)   # warm: maps, JIT-free, allocator
    torch.cuda.synchronize()
    strat = model.tune_kernel_shapes(t, opts, repeats=int(os.environ.get("REPS", "9")))
    save_strategy(out, strat)
    for r in strat.layers:
        if r.ctas or r.stage_kb:
            print(f"{r.layer_id:14s} ctas={r.ctas} stage_kb={r.stage_kb}")
    print("wrote", out)


if __name__ == "__main__":
    main()
