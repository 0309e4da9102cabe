"""Heavy-product kernel in isolation (cfg2-like shapes): time per launch for
the bitmap / count epilogues.

    python tools/mma_lab.py [rows] [ncols] [kpad]
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2002_12459_b200 import _native as nat  # noqa: E402


def main():
    rows = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
    ncols = int(sys.argv[2]) if len(sys.argv) > 2 else 500736
    kpad = int(sys.argv[3]) if len(sys.argv) > 3 else 128
    nat.load()
    g = torch.Generator(device="cuda").manual_seed(1)
    A = (torch.rand(rows, kpad, device="cuda", generator=g) < 0.05).to(torch.uint8)
    B = (torch.rand(ncols, kpad, device="cuda", generator=g) < 0.05).to(torch.uint8)
    wpr = ncols // 32
    out = torch.empty(rows * wpr, dtype=torch.int32, device="cuda")
    nnz = torch.zeros(1, dtype=torch.int64, device="cuda")
    z = torch.arange(ncols, device="cuda")
    b = z & 31
    prow = (z >> 5) * 16 + 2 * (b & 7) + ((b >> 3) >> 1)
    wgt = torch.where(((b >> 3) & 1) == 1, 128, 1).to(torch.int32)
    Bp = torch.zeros(ncols // 2, kpad, dtype=torch.int32, device="cuda")
    Bp.index_add_(0, prow, B.to(torch.int32) * wgt[:, None])
    Bp = Bp.to(torch.uint8)
    for mode, name in ((nat.MODE_BITMAP_PAIR, "bitmap_pair"), (nat.MODE_BITMAP_U8, "bitmap_u8"),
                       (nat.MODE_BITMAP, "bitmap_u16")):
        bb, brows = (Bp, ncols // 2) if mode == nat.MODE_BITMAP_PAIR else (B, ncols)
        for ctas in (0,):
            def run():
                nat.call("mmj_heavy_mma", nat.ptr(A), rows, nat.ptr(bb), brows, kpad, 0, kpad, 0, rows, mode, 0,
                         nat.ptr(out), wpr, nat.ptr(nnz), ctas, torch.cuda.current_stream().cuda_stream)
            for _ in range(3):
                run()
            if mode == nat.MODE_BITMAP_PAIR:
                ref = out.clone()
            elif mode == nat.MODE_BITMAP_U8:
                assert torch.equal(out, ref), "pair bitmap differs from the plain bitmap"
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            n = 10
            a.record()
            for _ in range(n):
                run()
            b.record()
            torch.cuda.synchronize()
            ms = a.elapsed_time(b) / n
            cells = rows * ncols
            tiles = (rows // 128) * (ncols // 256)   # per 32K output cells
            clk = 1.965e9
            print(f"{name} rows={rows} ncols={ncols} k={kpad}: "
                  f"{ms:.3f} ms  {cells / ms / 1e9:.2f} Tcell/s  {ms * 1e-3 * clk * 148 / tiles:.0f} clk/tile/SM  "
                  f"{2 * cells * kpad / ms / 1e9:.0f} TOPS  out {rows * wpr * 4 / ms / 1e6:.0f} GB/s")


if __name__ == "__main__":
    main()
