"""PCIe A/B for the e2e path (desc_transpose_host): which side of a banded transpose should
carry the strided (2-D) copy?  Banding by INPUT rows (the shipped pipeline) makes the H2D
copies contiguous and the D2H copies 2-D (cols rows of band*es bytes at pitch ld_out*es);
banding by OUTPUT rows (= input columns) makes the H2D 2-D and the D2H contiguous.

Times, for 8192^2 f32 split into bands of W bytes per strided row, the two directions running
concurrently on two streams (what the pipeline overlaps), each copy issued per band:
  contig : contiguous H2D || contiguous D2H  (the ceiling bench.py reports)
  d2h_2d : contiguous H2D || 2-D D2H          (current banding)
  h2d_2d : 2-D H2D        || contiguous D2H    (banding by output rows)
  python scripts/exp_pcie2d.py
"""
import torch
from cuda.bindings import runtime as rt

N = 8192
ES = 4


def run(mode, band, reps=3):
    nbytes = N * N * ES
    h_in = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    h_out = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    d_in = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    d_out = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    W = band * ES
    H2D, D2H = rt.cudaMemcpyKind.cudaMemcpyHostToDevice, rt.cudaMemcpyKind.cudaMemcpyDeviceToHost

    def cp2d(dst, dpitch, src, spitch, width, height, kind, stream):
        err, = rt.cudaMemcpy2DAsync(dst, dpitch, src, spitch, width, height, kind, stream.cuda_stream)
        assert err == rt.cudaError_t.cudaSuccess, err
    best = None
    for _ in range(reps):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        s1.wait_stream(torch.cuda.current_stream())
        s2.wait_stream(torch.cuda.current_stream())
        for k in range(N // band):
            lo = k * band * N * ES
            if mode == "h2d_2d":                 # input column stripe k: N rows of W bytes
                cp2d(d_in.data_ptr() + lo, W, h_in.data_ptr() + k * W, N * ES, W, N, H2D, s1)
            else:
                cp2d(d_in.data_ptr() + lo, W, h_in.data_ptr() + lo, W, W, N, H2D, s1)
            if mode == "d2h_2d":                 # output column stripe k: N rows of W bytes
                cp2d(h_out.data_ptr() + k * W, N * ES, d_out.data_ptr() + lo, W, W, N, D2H, s2)
            else:
                cp2d(h_out.data_ptr() + lo, W, d_out.data_ptr() + lo, W, W, N, D2H, s2)
        torch.cuda.current_stream().wait_stream(s1)
        torch.cuda.current_stream().wait_stream(s2)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        best = ms if best is None else min(best, ms)
    return 2 * nbytes / (best / 1e3) / 1e9


def main():
    for band in (256, 512, 1024, 2048):
        for mode in ("contig", "d2h_2d", "h2d_2d"):
            print(f"band {band:5d} rows ({band * ES:5d} B strided rows) {mode:7s} "
                  f"{run(mode, band):7.1f} GB/s (H2D + D2H bytes / time)", flush=True)


if __name__ == "__main__":
    main()
