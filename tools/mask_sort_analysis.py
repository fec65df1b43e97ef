"""How many (128-row tile, offset) blocks of a level-0 k3 map hold at least one
present neighbour, in the natural (coordinate) row order vs rows sorted by
their 27-bit presence mask (the TorchSparse++ bitmask reordering).  CPU only:
the oracle's map of one SemanticKITTI-shaped scan (test/analysis tool)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import load_scans  # noqa: E402
from oracle import sparseconv_oracle as O  # noqa: E402


def main(tile=128):
    c, _, b = load_scans(range(1))[0]
    c = np.asarray(c, np.int64)
    n = c.shape[0]
    pairs = O.kernel_map(c, b, c, 3, 1)
    mask = np.zeros(n, np.int64)
    for v, pr in enumerate(pairs):
        mask[pr[:, 1]] |= 1 << v
    present = ((mask[:, None] >> np.arange(len(pairs))) & 1).astype(bool)

    def live_blocks(order):
        m = present[order]
        nt = (n + tile - 1) // tile
        m = np.concatenate([m, np.zeros((nt * tile - n, m.shape[1]), bool)])
        return m.reshape(nt, tile, -1).any(1).mean()

    print(f"rows {n}, present (row, offset) fraction {present.mean():.3f}")
    print(f"live (tile, offset) blocks: natural order {live_blocks(np.arange(n)):.3f}, "
          f"mask-sorted {live_blocks(np.argsort(mask, kind='stable')):.3f}")


if __name__ == "__main__":
    main()
