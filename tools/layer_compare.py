"""Per-layer device time of MinkUNet (8 packed scans) under the staged and the
fused dataflow (StageTimer, CUDA events), to derive the ``auto`` rule."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2204_10319_b200 as sc  # noqa: E402
from bench import load_scans, pack  # noqa: E402
from paper_2204_10319_b200.minkunet import EngineMinkUNet  # noqa: E402


def run(model, cd, fd, b, df, reps=5):
    timer = sc.StageTimer()
    for i in range(reps + 2):
        t = sc.SparseTensor(cd, fd, 1, b, 8, validate=False)
        t = sc.quantize_features(t, sc.PrecisionMode.FP16_STORAGE)
        opts = sc.ExecOptions(index_kind="hash", dataflow=df, timer=timer if i >= 2 else None)
        model.forward(t, opts)
    per = {}
    for (layer, stage), v in timer.samples.items():
        if stage != "mapping":
            per[layer] = per.get(layer, 0.0) + v / reps
    return per


def main():
    c, f, b = pack(load_scans(range(8)))
    cd = torch.from_numpy(c.astype(np.int32)).cuda()
    fd = torch.from_numpy(f).cuda()
    model = EngineMinkUNet(1.0, 4, 0)
    shapes = {l["name"]: l for l in model.table}
    st = run(model, cd, fd, b, "staged")
    fu = run(model, cd, fd, b, "fused")
    tot_s = tot_f = tot_b = 0.0
    for name in st:
        l = shapes.get(name, {})
        s, fz = st[name] * 1e3, fu.get(name, float("nan")) * 1e3
        tot_s += s
        tot_f += fz if fz == fz else s
        tot_b += min(s, fz) if fz == fz else s
        print(f"{name:14s} {str(l.get('ci')):>4s}->{str(l.get('co')):<4s} k{l.get('k')} "
              f"staged {s:7.3f} fused {fz:7.3f}  {'F' if fz < s else 'S'}")
    print(f"total staged {tot_s:.2f} fused {tot_f:.2f} best-of {tot_b:.2f} ms")


if __name__ == "__main__":
    main()
