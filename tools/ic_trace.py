"""Per-stage timeline of the fused conv (trace build: `make trace`):
issue -> full latency (the gather of a stage), MMA-side waits, stage period.
    SCB_LIB_NAME=libsparseconv_b200_trace.so CIN=96 COUT=96 python tools/ic_trace.py"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2204_10319_b200 as sc  # noqa: E402
from paper_2204_10319_b200 import _native as nat  # noqa: E402
from paper_2204_10319_b200.core import CoordinateSet  # noqa: E402
from paper_2204_10319_b200.mapping import reorder_by_presence  # noqa: E402
from bench import load_scans, pack  # noqa: E402

CTAS, STAGES = 4, 512


def main():
    assert "trace" in os.environ.get("SCB_LIB_NAME", ""), "needs the trace build"
    c, f, b = pack(load_scans(range(8)))
    cin, cout = int(os.environ.get("CIN", "96")), int(os.environ.get("COUT", "96"))
    rng = np.random.default_rng(0)
    cset = CoordinateSet(torch.from_numpy(c.astype(np.int32)).cuda(), b, 8)
    cset = reorder_by_presence(cset, 3, "hash")
    feats = torch.from_numpy(rng.standard_normal((c.shape[0], cin)).astype(np.float16)).cuda()
    t = sc.SparseTensor._wrap(feats, 1, b, 8, cset)
    w = sc.WeightTensor(rng.normal(0, 0.05, (27, cin, cout)).astype(np.float32), 3, 3)
    spec = sc.LayerSpec(3, 1, cin, cout)
    shape = tuple(int(x) for x in os.environ.get("SHAPE", "0:0").split(":"))
    opts = sc.ExecOptions(dataflow="fused", index_kind="hash", layer_label="L",
                          kernel_shapes={"L": shape})
    lib = nat.load()
    lib.scb_ic_trace_read.argtypes = [ctypes.c_void_p, ctypes.c_int64]
    for _ in range(5):
        sc.sparse_conv_forward(t, w, spec, None, None, opts)
    torch.cuda.synchronize()
    lib.scb_ic_trace_clear()
    sc.sparse_conv_forward(t, w, spec, None, None, opts)
    torch.cuda.synchronize()
    buf = np.zeros(CTAS * STAGES * 6, dtype=np.int64)
    lib.scb_ic_trace_read(buf.ctypes.data, buf.size)
    tr = buf.reshape(CTAS, STAGES, 6)
    for cta in [int(x) for x in os.environ.get("TRACE_CTAS", "0,1").split(",")]:
        x = tr[cta]
        n = int(np.count_nonzero(x[:, 2]))
        x = x[:n].astype(np.float64)
        x -= x[0, 0]
        lat = x[:, 3] - x[:, 0]          # copies issued -> A full (gather latency)
        bwait = x[:, 1] - x[:, 3]        # A full -> B full (weights later than rows)
        work = x[:, 2] - x[:, 1]         # full -> committed (issue time)
        fence = x[:, 4] - x[:, 1]        # full -> past the proxy fence
        issue = x[:, 5] - x[:, 4]        # the stage's MMA instructions
        mma_gap = np.diff(x[:, 1])       # MMA-side period
        commit_to_next_issue = x[2:, 0] - x[:-2, 2]  # (2-stage ring) slot freed -> reissue
        print(f"CTA {cta}: {n} stages over {x[-1, 2]:.0f} cycles = {x[-1, 2] / n:.0f} cyc/stage")
        for name, v in (("issue->A full (gather latency)", lat), ("A full->B full", bwait),
                        ("full->commit", work), ("full->fenced", fence), ("MMA issue", issue), ("full->full (MMA period)", mma_gap),
                        ("commit(s)->issue(s+2)", commit_to_next_issue)):
            q = np.percentile(v[5:], [10, 50, 90]) if v.size > 10 else v
            print(f"   {name:32s} p10 {q[0]:7.0f}  p50 {q[1]:7.0f}  p90 {q[2]:7.0f}")
        print("   first stages (issue, full, commit):")
        for i in range(10, 16):
            print(f"     {i:3d} {x[i, 0]:8.0f} {x[i, 3]:8.0f} {x[i, 1]:8.0f} {x[i, 2]:8.0f}")


if __name__ == "__main__":
    main()
