"""cProfile the host side of the MinkUNet bench forward (8 packed scans)."""
import cProfile
import os
import pstats
import sys
import time

import numpy as np
import torch

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

    for _ in range(3):
        step()
    torch.cuda.synchronize()
    pr = cProfile.Profile()
    t0 = time.perf_counter()
    pr.enable()
    for _ in range(5):
        step()
    pr.disable()
    torch.cuda.synchronize()
    print(f"wall {1e3 * (time.perf_counter() - t0) / 5:.2f} ms/step")
    st = pstats.Stats(pr)
    st.sort_stats("tottime").print_stats(25)


if __name__ == "__main__":
    main()
