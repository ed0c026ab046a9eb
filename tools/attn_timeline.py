"""Per-block timeline of the CTA-pair attention kernel (attention_kernel_2sm),
from the TN_ATTN_DBG probe: run e.g.

    TN_ATTN_DBG=gpurun_out/attn_dbg.txt python tools/attn_bench.py --reps 1 --runs 3
    python tools/attn_timeline.py gpurun_out/attn_dbg.txt

Each launch appends one line of 4096 clock64 stamps (cluster 0, its first
item, leader CTA): the MMA issuer's waits for P_t,j (halves A and B) and, for
one softmax warp per tile, the S_t,j wait, TMEM load, row max, the two P
hand-offs. Prints the steady-state means of the last launch."""
import sys

import numpy as np


def main(path):
    d = np.array([int(x) for x in open(path).read().strip().splitlines()[-1].split()], dtype=np.int64)
    iss = d[:512].reshape(2, 64, 4)
    sm = d[512:1536].reshape(2, 64, 8)
    for t in range(2):
        nk = int((sm[t, :, 5] > 0).sum())
        js = range(4, nk - 2)

        def f(a, b, arr=sm):
            return float(np.mean([arr[t, j, b] - arr[t, j, a] for j in js]))

        period = float(np.mean([sm[t, j + 1, 1] - sm[t, j, 1] for j in js]))
        print(f"tile {t}: {nk} blocks, period {period:.0f} clk | softmax: wait S {f(0, 1):.0f}, TMEM load {f(1, 2):.0f}, "
              f"max {f(2, 3):.0f}, 2^x + P half A {f(3, 4):.0f}, half B {f(4, 5):.0f} | issuer: wait P_A {f(0, 1, iss):.0f}, "
              f"P_B {f(1, 2, iss):.0f}")


if __name__ == "__main__":
    main(sys.argv[1])
