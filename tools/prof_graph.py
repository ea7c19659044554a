"""Device time of one tl_matmul launch, host overhead removed: the launches are captured in a
CUDA graph and the weight copies rotate over > 2x L2 so every launch streams from HBM.

    python tools/prof_graph.py FMT LAYER M [PATH] [FMT LAYER M [PATH] ...]
"""
import sys

import torch

sys.path.insert(0, ".")
import paper_2504_12984_b200 as P  # noqa: E402
import workloads as wl  # noqa: E402


def run(fmt, layer, M, path):
    K, N = wl.LLAMA33_70B[layer] if layer in wl.LLAMA33_70B else map(int, layer.split("x"))
    w = P.wtype(fmt)
    b = int(fmt[1])
    zp = fmt[0] == "u"
    byts = K * N * b / 8 + (K // 128) * N * 2 * (1 + zp) + 2 * M * (K + N)
    nc = max(1, int(-(-300e6 // byts)))
    copies = []
    for c in range(nc):
        codes = wl.gen_codes_torch(fmt, K, N, c + 1)
        wt = P.tl_transform_weights(w, K, N, P.tl_pack(w, K, N, codes))
        del codes
        copies.append((wt, wl.gen_scales_torch(fmt, K, N, 128, c + 1), wl.gen_zeros_torch(fmt, K, N, 128, c + 1)))
    A = wl.gen_activations_torch(M, K, 1)
    Y = torch.empty((M, N), dtype=torch.float16, device="cuda")
    ws = P.alloc_workspace(w, M, N, K, 128)
    reps = max(2 * nc, 8)

    def launches():
        for i in range(reps):
            wt, s, z = copies[i % nc]
            P.tl_matmul_ex(w, M, N, K, 128, A, wt, s, z, Y, ws, path=path)

    launches()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        launches()
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    R = 5
    for _ in range(R):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / (R * reps) * 1e3
    print(f"{fmt:7s} {layer:8s} M={M:<3d} path={path} us={us:7.2f} GB/s={byts / us / 1e3:6.0f} "
          f"TFLOP/s={2 * M * N * K / us / 1e6:6.1f}", flush=True)
    del copies, g


if __name__ == "__main__":
    a = sys.argv[1:]
    i = 0
    while i < len(a):
        fmt, layer, M = a[i], a[i + 1], int(a[i + 2])
        path = 0
        if i + 3 < len(a) and a[i + 3].isdigit():
            path = int(a[i + 3])
            i += 1
        run(fmt, layer, M, path)
        i += 3
