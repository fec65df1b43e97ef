"""Why does the per-step D2H of the logits add its own duration to the
step?  Variants of the device-resident loop plus one D2H per step."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2204_10319_b200 as sc  # noqa: E402
from bench import load_scans, pack  # noqa: E402
from paper_2204_10319_b200.minkunet import EngineMinkUNet  # noqa: E402


def main():
    coords, feats, boundary = pack(load_scans(range(8)))
    model = EngineMinkUNet(1.0, 4, 0)
    d_c = torch.from_numpy(coords.astype(np.int32)).cuda()
    d_f = torch.from_numpy(feats).cuda()

    def fwd():
        t = sc.SparseTensor(d_c, d_f, 1, boundary, 8, validate=False)
        t = sc.quantize_features(t, sc.PrecisionMode.FP16_STORAGE)
        return model.forward(t, sc.ExecOptions(index_kind="hash", dataflow="auto"))

    o = fwd()
    torch.cuda.synchronize()
    f = o.features
    full = f.as_strided((f.shape[0], f.stride(0)), (f.stride(0), 1))
    h_big = torch.empty(tuple(full.shape), dtype=full.dtype).pin_memory()
    h_small = torch.empty((1, full.shape[1]), dtype=full.dtype).pin_memory()
    lo_prio = torch.cuda.Stream()
    hi_prio = torch.cuda.Stream(priority=-1)
    staging = torch.empty_like(full)

    def loop(kind, steps=20):
        evs = []
        for _ in range(5 + steps):
            o = fwd()
            ff = o.features
            src = ff.as_strided((ff.shape[0], ff.stride(0)), (ff.stride(0), 1))
            done = torch.cuda.current_stream().record_event()
            if kind == "none":
                pass
            elif kind == "small":
                lo_prio.wait_event(done)
                with torch.cuda.stream(lo_prio):
                    h_small.copy_(src[:1], non_blocking=True)
            elif kind in ("big", "big_hi"):
                s = lo_prio if kind == "big" else hi_prio
                s.wait_event(done)
                with torch.cuda.stream(s):
                    h_big.copy_(src, non_blocking=True)
            elif kind == "chunks":
                lo_prio.wait_event(done)
                with torch.cuda.stream(lo_prio):
                    n = src.shape[0]
                    for i in range(8):
                        a, b = n * i // 8, n * (i + 1) // 8
                        h_big[a:b].copy_(src[a:b], non_blocking=True)
            elif kind == "staged":
                staging.copy_(src)  # D2D on the compute stream
                d2 = torch.cuda.current_stream().record_event()
                lo_prio.wait_event(d2)
                with torch.cuda.stream(lo_prio):
                    h_big.copy_(staging, non_blocking=True)
            elif kind == "same_stream":
                h_big.copy_(src, non_blocking=True)
            ev = torch.cuda.Event(enable_timing=True)
            ev.record()
            evs.append(ev)
        torch.cuda.synchronize()
        lo_prio.synchronize()
        hi_prio.synchronize()
        ms = evs[4].elapsed_time(evs[-1]) / steps
        print(f"{kind:12s} {ms:7.3f} ms/step", flush=True)

    for k in ("none", "small", "big", "big_hi", "chunks", "staged", "same_stream", "none", "big"):
        loop(k)


if __name__ == "__main__":
    main()
