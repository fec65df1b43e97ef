"""Time one MinkUNet-like level-0 layer (8 packed scans) per dataflow and per
SCB_IMPLICIT_DEBUG variant; prints ms per launch (CUDA events)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2204_10319_b200 as sc  # noqa: E402
from bench import load_scans, pack  # noqa: E402


def main():
    c, f, b = pack(load_scans(range(int(os.environ.get("NSCANS", "8")))))
    lv = int(os.environ.get("LEVEL", "0"))
    if lv:  # emulate pyramid level lv: coordinates // 2^lv, unique
        cc = c.astype(np.int64).copy()
        cc[:, 1:] >>= lv
        c = np.unique(cc, axis=0).astype(c.dtype)
    cin = int(os.environ.get("CIN", "32"))
    cout = int(os.environ.get("COUT", "32"))
    k = int(os.environ.get("K", "3"))
    s = int(os.environ.get("S", "1"))
    rng = np.random.default_rng(0)
    feats = torch.from_numpy(rng.standard_normal((c.shape[0], cin)).astype(np.float16)).cuda()
    t = sc.SparseTensor(torch.from_numpy(c.astype(np.int32)).cuda(), feats, 1, b, 8, validate=False)
    w = sc.WeightTensor(rng.normal(0, 0.05, (k ** 3, cin, cout)).astype(np.float32), k, 3)
    spec = sc.LayerSpec(k, s, cin, cout)
    for df in os.environ.get("DATAFLOWS", "staged,fused").split(","):
        opts = sc.ExecOptions(dataflow=df, index_kind="hash")
        # warm (map build + clock ramp: >= 0.5 s of back-to-back launches)
        t_end = time.time() + 0.5
        while time.time() < t_end:
            out = sc.sparse_conv_forward(t, w, spec, None, None, opts)
            torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20):
            out = sc.sparse_conv_forward(t, w, spec, None, None, opts)
        e1.record()
        torch.cuda.synchronize()
        print(f"{df:7s} dbg={os.environ.get('SCB_IMPLICIT_DEBUG', '0')} N={c.shape[0]} "
              f"C={cin}->{cout} K={k}: {e0.elapsed_time(e1) / 20:.3f} ms/layer", flush=True)


if __name__ == "__main__":
    main()
