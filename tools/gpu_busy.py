"""GPU busy time vs wall time of one bench step (torch.profiler kernel
timeline, warm), plus the top kernels.  Diagnoses host-bound vs GPU-bound."""
import os
import sys

import numpy as np
import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2204_10319_b200 as sc  # noqa: E402
from bench import load_scans, pack  # noqa: E402
from paper_2204_10319_b200.minkunet import EngineMinkUNet  # noqa: E402


def main():
    c, f, b = pack(load_scans(range(8)))
    cd = torch.from_numpy(c.astype(np.int32)).cuda()
    fd = torch.from_numpy(f).cuda()
    model = EngineMinkUNet(1.0, 4, 0)
    df = os.environ.get("DATAFLOW", "auto")

    def step():
        t = sc.SparseTensor(cd, fd, 1, b, 8, validate=False)
        t = sc.quantize_features(t, sc.PrecisionMode.FP16_STORAGE)
        return model.forward(t, sc.ExecOptions(index_kind="hash", dataflow=df))

    for _ in range(4):
        step()
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
        for _ in range(3):
            step()
        torch.cuda.synchronize()
    evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
    kern = [e for e in evs if e.time_range.elapsed_us() > 0]
    start = min(e.time_range.start for e in kern)
    end = max(e.time_range.end for e in kern)
    # union of kernel intervals
    iv = sorted((e.time_range.start, e.time_range.end) for e in kern)
    busy, cur_s, cur_e = 0, None, None
    for s, e in iv:
        if cur_e is None or s > cur_e:
            if cur_e is not None:
                busy += cur_e - cur_s
            cur_s, cur_e = s, e
        else:
            cur_e = max(cur_e, e)
    busy += cur_e - cur_s
    print(f"span {(end - start) / 3e3:.2f} ms/step, GPU busy {busy / 3e3:.2f} ms/step "
          f"({100 * busy / (end - start):.0f}%)")
    # the largest idle gaps of the last profiled step, with the kernels around them
    seq = sorted(kern, key=lambda e: e.time_range.start)
    gaps = []
    for a, b in zip(seq, seq[1:]):
        g = b.time_range.start - a.time_range.end
        if g > 0:
            gaps.append((g, a.name[:40], b.name[:40]))
    gaps.sort(reverse=True)
    for g, a, b in gaps[:12]:
        print(f"gap {g:8.1f} us  after {a}  before {b}")
    print(f"gaps > 5 us: {sum(1 for g in gaps if g[0] > 5)}, total {sum(g[0] for g in gaps) / 3e3:.3f} ms/step")
    agg = {}
    for e in kern:
        k = e.name[:60]
        agg[k] = agg.get(k, 0) + e.time_range.elapsed_us()
    for k, v in sorted(agg.items(), key=lambda x: -x[1])[:15]:
        print(f"{v / 3e3:8.3f} ms/step  {k}")


if __name__ == "__main__":
    main()
