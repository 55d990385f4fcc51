"""Time the column-pivoted QR pieces on the device (CUDA events): the
dgeqp3-rule pivot kernel and the full column_pivoted_qr, for UTV-core sizes.

    python tools/cpqr_probe.py
"""
import sys

import numpy as np
import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2103_07245_b200 import device as D  # noqa: E402
from paper_2103_07245_b200.linalg import cpqr_device  # noqa: E402


def main():
    dev = torch.device("cuda", 0)
    ctx = D.context(dev)
    rng = np.random.default_rng(0)
    for n in (64, 256, 512, 1024):
        m = rng.standard_normal((n, n)) @ np.diag(np.exp(-np.arange(n) / (n / 10))) @ rng.standard_normal((n, n))
        t = D.as_kernel_operand(torch.from_numpy(m).to(dev))
        for _ in range(2):
            D.cpqr_pivots(ctx, t)
            cpqr_device(ctx, t)
        torch.cuda.synchronize()
        e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        e[0].record()
        for _ in range(5):
            D.cpqr_pivots(ctx, t)
        e[1].record()
        for _ in range(5):
            cpqr_device(ctx, t)
        e[2].record()
        torch.cuda.synchronize()
        piv = e[0].elapsed_time(e[1]) / 5
        full = e[1].elapsed_time(e[2]) / 5
        print(f"n={n}: pivots {piv:.3f} ms ({1e3 * piv / n:.2f} us/step), column_pivoted_qr {full:.3f} ms", flush=True)


if __name__ == "__main__":
    main()
