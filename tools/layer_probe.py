"""One fused k3 layer of the bench's level 0 (8 packed scans, rows
relabelled by presence mask exactly as EngineMinkUNet does), timed with CUDA
events, plus the work it executes: live (tile, offset) blocks, MMAs,
useful / executed FLOPs and cycles per MMA at the measured clock.

    CIN=96 COUT=96 LEVEL=0 REORDER=1 python tools/layer_probe.py
Under ncu, filter on implicit_conv_f16_kernel and skip the warm-up launches."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2204_10319_b200 as sc  # noqa: E402
from paper_2204_10319_b200.core import CoordinateSet  # noqa: E402
from paper_2204_10319_b200.mapping import reorder_by_presence  # noqa: E402
from bench import load_scans, pack  # noqa: E402


def main():
    c, f, b = pack(load_scans(range(int(os.environ.get("NSCANS", "8")))))
    lv = int(os.environ.get("LEVEL", "0"))
    if lv:  # pyramid level lv: coordinates // 2^lv, unique
        cc = c.astype(np.int64).copy()
        cc[:, 1:] >>= lv
        c = np.unique(cc, axis=0)
        b = tuple(-(-x // (1 << lv)) for x in b)
    cin, cout = int(os.environ.get("CIN", "96")), int(os.environ.get("COUT", "96"))
    reps = int(os.environ.get("REPS", "20"))
    rng = np.random.default_rng(0)
    coords = torch.from_numpy(c.astype(np.int32)).cuda()
    cset = CoordinateSet(coords, b, 8)
    if os.environ.get("REORDER", "1") == "1":
        cset = reorder_by_presence(cset, 3, "hash")
    feats = torch.from_numpy(rng.standard_normal((c.shape[0], cin)).astype(np.float16)).cuda()
    t = sc.SparseTensor._wrap(feats, 1, b, 8, cset)
    w = sc.WeightTensor(rng.normal(0, 0.05, (27, cin, cout)).astype(np.float32), 3, 3)
    spec = sc.LayerSpec(3, 1, cin, cout)
    opts = sc.ExecOptions(dataflow="fused", index_kind="hash")
    out = sc.sparse_conv_forward(t, w, spec, None, None, opts)
    kmap = cset.maps[(3, 1, -1)][1]
    masks = kmap.tile_masks().cpu().numpy().astype(np.uint32)
    live = int(sum(bin(int(m)).count("1") for m in masks))
    n = c.shape[0]
    useful = 2.0 * kmap.total * cin * cout
    kc = 16 * ((cin + 15) // 16)
    mmas = live * kc // 16
    executed = 2.0 * live * 128 * kc * cout
    t_end = time.time() + (0.0 if os.environ.get("NOWARM") else 0.5)
    while time.time() < t_end:
        out = sc.sparse_conv_forward(t, w, spec, None, None, opts)
        torch.cuda.synchronize()
    shapes = [tuple(int(x) for x in sh.split(":")) for sh in os.environ.get("SHAPES", "").split(",")
              if sh]
    for sh in shapes:  # launch-shape sweep: (CTAs per SM, stage KB)
        o2 = sc.ExecOptions(dataflow="fused", index_kind="hash", layer_label="probe",
                            kernel_shapes={"probe": sh})
        sc.sparse_conv_forward(t, w, spec, None, None, o2)
        a, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(reps):
            sc.sparse_conv_forward(t, w, spec, None, None, o2)
        b_.record()
        torch.cuda.synchronize()
        print(f"  shape ctas={sh[0]} stage_kb={sh[1]}: {a.elapsed_time(b_) / reps:.4f} ms", flush=True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        out = sc.sparse_conv_forward(t, w, spec, None, None, opts)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    sm = torch.cuda.get_device_properties(0).multi_processor_count
    mhz = float(os.environ.get("MHZ", "1965"))
    cyc = ms * 1e-3 * mhz * 1e6 * sm / max(mmas, 1)
    print(f"N={n} C={cin}->{cout} L{lv} reorder={os.environ.get('REORDER', '1')} "
          f"l1={os.environ.get('SCB_IC_L1', '0')}: {ms:.4f} ms  "
          f"tiles={masks.shape[0]} live_blocks={live} ({live / masks.shape[0] / 27:.3f})  "
          f"|M|/(27N)={kmap.total / 27 / n:.3f}  useful {useful / ms / 1e9:.0f} TF/s  "
          f"executed {executed / ms / 1e9:.0f} TF/s  {cyc:.0f} SM-cycles per K16 MMA", flush=True)
    del out


if __name__ == "__main__":
    main()
