"""Host<->device copy bandwidth on the GPU box (pinned memory), for the e2e leg.

Measures contiguous and pitched (layout-R column chunk) copies, one direction
at a time and both directions at once on two streams.
    python tools/pcie_bench.py
"""
import time

import torch
from cuda.bindings import runtime as rt


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    return best


def main():
    nbytes = 128 << 20
    h_in = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    h_out = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    d_a = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    d_b = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

    def h2d():
        with torch.cuda.stream(s1):
            d_a.copy_(h_in, non_blocking=True)

    def d2h():
        with torch.cuda.stream(s2):
            h_out.copy_(d_b, non_blocking=True)

    def both():
        h2d()
        d2h()

    for name, fn, b in (("h2d contiguous", h2d, nbytes), ("d2h contiguous", d2h, nbytes),
                        ("h2d+d2h concurrent", both, 2 * nbytes)):
        t = timed(fn)
        print(f"{name:28s} {b / t / 1e9:7.1f} GB/s  ({t * 1e3:.2f} ms)")

    # pitched: 4096 rows x 32 KB, copy a column chunk of w bytes per row
    rows, pitch = 4096, 32768
    hF = h_in[: rows * pitch].view(rows, pitch)
    hX = h_out[: rows * pitch].view(rows, pitch)
    for w in (2048, 4096, 8192, 16384):
        dA = d_a[: rows * w].view(rows, w)
        dB = d_b[: rows * w].view(rows, w)

        def p_h2d():
            for c in range(pitch // w):
                rt.cudaMemcpy2DAsync(dA.data_ptr(), w, hF.data_ptr() + c * w, pitch, w, rows,
                                     rt.cudaMemcpyKind.cudaMemcpyHostToDevice, s1.cuda_stream)

        def p_both():
            for c in range(pitch // w):
                rt.cudaMemcpy2DAsync(dA.data_ptr(), w, hF.data_ptr() + c * w, pitch, w, rows,
                                     rt.cudaMemcpyKind.cudaMemcpyHostToDevice, s1.cuda_stream)
                rt.cudaMemcpy2DAsync(hX.data_ptr() + c * w, pitch, dB.data_ptr(), w, w, rows,
                                     rt.cudaMemcpyKind.cudaMemcpyDeviceToHost, s2.cuda_stream)

        t = timed(p_h2d)
        t2 = timed(p_both)
        print(f"pitched w={w:5d} h2d {rows * pitch / t / 1e9:7.1f} GB/s   "
              f"h2d+d2h {2 * rows * pitch / t2 / 1e9:7.1f} GB/s")


if __name__ == "__main__":
    main()
