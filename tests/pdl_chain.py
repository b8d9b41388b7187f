"""Helper for tests/test_gpu_parity.py::test_pdl_chain_bitwise (run in a subprocess so CONV2D_PDL, read once per
process, can differ): a chain of convs where each consumes the previous output, captured into one CUDA graph,
every algorithm / path on the way; prints the sha256 of every output."""
import hashlib
import sys

import torch

sys.path.insert(0, sys.argv[1])
from paper_1904_04174_b200 import conv2d as C  # noqa: E402
from paper_1904_04174_b200 import synth  # noqa: E402

# (C_in -> F, window, stride, algo): dense 1x1, im2col 3x3 (split / halo paths by shape), Winograd, direct,
# tiled, strided 1x1, 7x7 stem-like; every output is the next conv's input
CHAIN = [(64, 64, 3, 1, C.ALGO_IMPLICIT_GEMM), (64, 128, 1, 1, C.ALGO_MATMUL_1X1),
         (128, 128, 3, 1, C.ALGO_WINOGRAD_F4X4_3X3), (128, 64, 3, 1, C.ALGO_WINOGRAD_F2X2_3X3),
         (64, 64, 3, 1, C.ALGO_DIRECT), (64, 64, 3, 1, C.ALGO_TILED), (64, 256, 1, 2, C.ALGO_IMPLICIT_GEMM),
         (256, 256, 3, 1, C.ALGO_IMPLICIT_GEMM), (256, 64, 1, 1, C.ALGO_MATMUL_1X1)]


def main():
    n, h = 4, 28
    x = torch.empty(n * h * h * CHAIN[0][0], device="cuda")
    C.conv2d_synth_fill(x, x.numel(), synth.stream_key(synth.SEED, 4000, 0), 0, 0)
    bufs, plan = [x], []
    hh = h
    for i, (c, f, k, s, a) in enumerate(CHAIN):
        p = C.Params(n, hh, hh, c, f, k, k, s, s, C.PAD_SAME)
        (nn, ho, wo, ff), _ = C.conv2d_output_shape(p)
        w = torch.empty(k * k * c * f, device="cuda")
        C.conv2d_synth_fill(w, w.numel(), synth.stream_key(synth.SEED, 4000 + i, 1), 0, 0)
        w.mul_(1.0 / (k * k * c) ** 0.5)  # keep activations O(1) along the chain
        y = torch.empty(nn * ho * wo * ff, device="cuda")
        need = C.conv2d_query_workspace(p, a)
        ws = torch.empty(max(need, 16), dtype=torch.uint8, device="cuda")
        plan.append((p, a, bufs[-1], w, y, ws, need))
        bufs.append(y)
        hh = ho
    s = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s, capture_error_mode="thread_local"):
        for p, a, xin, w, y, ws, need in plan:
            C.conv2d_forward(p, a, xin, w, y, ws, need, s)
    for _ in range(3):
        for y in bufs[1:]:
            y.fill_(float("nan"))
        g.replay()
        torch.cuda.synchronize()
    for y in bufs[1:]:
        print(hashlib.sha256(y.cpu().numpy().tobytes()).hexdigest())


if __name__ == "__main__":
    main()
