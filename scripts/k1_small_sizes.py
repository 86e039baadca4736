"""K1 at C5's small sizes: the TMA kernel (variant 1, the default) against the
SIMT kernel (variant 0), each launch cold and clean (read flush), CUDA events.

    python scripts/k1_small_sizes.py
"""

import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2108_05818_b200 import _native as N  # noqa: E402
from paper_2108_05818_b200 import kernels as K  # noqa: E402
from paper_2108_05818_b200 import microbench as MB  # noqa: E402


def main():
    flush = MB.L2Flush()
    peak = MB.measured_peak_gbs()
    lib = N.load()
    for lg in (20, 21, 22, 23, 24, 25, 26):
        n = 1 << lg
        p16 = (torch.randn(n, device="cuda") * 1e-3).half()
        p32 = torch.randn(n, device="cuda") * 0.02
        m, v = torch.zeros(n, device="cuda"), torch.zeros(n, device="cuda")
        hyper = K.AdamHyper(lr=1e-4)
        st = K.StepState("cuda")
        st.sumsq().fill_(1.0)
        K.adam_prepare(st, hyper)
        row = {"n": n}
        for var in (0, 1):
            lib.cs_adam_variant(var)
            ms = MB.time_launch(lambda: K.adam_chunks([(p16, p32, m, v, n)], hyper, st), 20,
                                flush)
            row["variant%d_ms" % var] = round(ms, 5)
            row["variant%d_frac" % var] = round(28 * n / (ms * 1e-3) / 1e9 / peak, 4)
        lib.cs_adam_variant(1)
        print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main()
