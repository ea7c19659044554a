"""Device time of one tl_matmul_ex at several split-K grids: fmt layer M path grid1 grid2 ..."""
import sys
sys.path.insert(0, ".")
import torch
import paper_2504_12984_b200 as P
import workloads as wl
fmt, layer, M, path = sys.argv[1], sys.argv[2], int(sys.argv[3]), int(sys.argv[4])
grids = [int(x) for x in sys.argv[5:]]
K, N = wl.LLAMA33_70B[layer] if layer in wl.LLAMA33_70B else wl.QWEN25_32B[layer]
w = P.wtype(fmt)
wt = P.tl_transform_weights(w, K, N, P.tl_pack(w, K, N, wl.gen_codes_torch(fmt, K, N, 1)))
s = wl.gen_scales_torch(fmt, K, N, 128, 1); z = wl.gen_zeros_torch(fmt, K, N, 128, 1)
A = wl.gen_activations_torch(M, K, 1); Y = torch.empty((M, N), dtype=torch.float16, device="cuda")
ws = P.alloc_workspace(w, M, N, K, 128)
for g in grids:
    for _ in range(3):
        P.tl_matmul_ex(w, M, N, K, 128, A, wt, s, z, Y, ws, path=path, splits=g)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        P.tl_matmul_ex(w, M, N, K, 128, A, wt, s, z, Y, ws, path=path, splits=g)
    e1.record(); torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / 20 * 1e3
    print(f"{fmt} {layer} M={M} path={path} grid={g} us={us:.2f} TFLOP/s={2*M*N*K/us/1e6:.1f}", flush=True)
