"""Sweep the implicit-conv launch knobs (CTAs per SM, offsets per stage) per
channel shape on one MinkUNet-like level-0 map (8 packed scans)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2204_10319_b200 as sc  # noqa: E402
from bench import load_scans, pack  # noqa: E402


CONFIGS = [(1, 2, -1, 32, 1), (1, 2, -1, 48, 1), (1, 2, -1, 32, 0), (1, 2, -1, 48, 0),
           (1, 1, -1, 64, 1), (1, 1, -1, 64, 0), (2, 1, -1, 96, 1), (2, 1, -1, 96, 0),
           (2, 2, -1, 32, 1)]


def timeit(fn, n=20):
    t_end = time.time() + 0.3
    while time.time() < t_end:
        fn()
        torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


def main():
    c, f, b = pack(load_scans(range(8)))
    rng = np.random.default_rng(0)
    coords = torch.from_numpy(c.astype(np.int32)).cuda()
    shapes = [tuple(map(int, s.split("x"))) for s in
              os.environ.get("SHAPES", "16x32,32x32,64x64,96x96,128x96,64x128,128x128,256x256").split(",")]
    for cin, cout in shapes:
        feats = torch.from_numpy(rng.standard_normal((c.shape[0], cin)).astype(np.float16)).cuda()
        t = sc.SparseTensor(coords, feats, 1, b, 8, validate=False)
        w = sc.WeightTensor(rng.normal(0, 0.05, (27, cin, cout)).astype(np.float32), 3, 3)
        spec = sc.LayerSpec(3, 1, cin, cout)
        res = {}
        o_st = sc.ExecOptions(dataflow="staged", index_kind="hash")
        res["staged"] = timeit(lambda: sc.sparse_conv_forward(t, w, spec, None, None, o_st))
        o_f = sc.ExecOptions(dataflow="fused", index_kind="hash")
        ref = sc.sparse_conv_forward(t, w, spec, None, None, o_st).features.float()
        for T, ctas, lag, kb, P in CONFIGS:
            os.environ.update(SCB_IC_T=str(T), SCB_IMPLICIT_CTAS=str(ctas), SCB_IC_COAL=str(P),
                              SCB_IMPLICIT_LAG=str(lag), SCB_IC_STAGE_KB=str(kb))
            try:
                ms = timeit(lambda: sc.sparse_conv_forward(t, w, spec, None, None, o_f))
                got = sc.sparse_conv_forward(t, w, spec, None, None, o_f).features.float()
                err = float((got - ref).norm() / ref.norm())
                res[f"T{T}c{ctas}C{P}k{kb}"] = ms if err < 1e-2 else float("nan")
            except Exception:  # stage does not fit
                pass
        for k in ("SCB_IC_T", "SCB_IMPLICIT_CTAS", "SCB_IC_COAL", "SCB_IMPLICIT_LAG", "SCB_IC_STAGE_KB"):
            os.environ.pop(k, None)
        best = min((v, k) for k, v in res.items() if v == v)
        print(f"{cin}->{cout}: best {best[1]} {best[0]:.3f} | " +
              " ".join(f"{k}={v:.3f}" for k, v in res.items()), flush=True)


if __name__ == "__main__":
    main()
