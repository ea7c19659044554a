import sys, torch
sys.path.insert(0, '.')
import paper_2504_12984_b200 as P, workloads as wl
fmt, layer, M = sys.argv[1], sys.argv[2], int(sys.argv[3])
path = int(sys.argv[4]) if len(sys.argv) > 4 else 0
K, N = wl.LLAMA33_70B[layer]
w = P.wtype(fmt)
codes = wl.gen_codes_torch(fmt, K, N, 1)
wt = P.tl_transform_weights(w, K, N, P.tl_pack(w, K, N, codes)); del codes
s = wl.gen_scales_torch(fmt, K, N, 128, 1); z = wl.gen_zeros_torch(fmt, K, N, 128, 1)
A = wl.gen_activations_torch(M, K, 1); Y = torch.empty((M, N), dtype=torch.float16, device='cuda')
ws = P.alloc_workspace(w, M, N, K, 128)
for _ in range(5): P.tl_matmul_ex(w, M, N, K, 128, A, wt, s, z, Y, ws, path=path)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20): P.tl_matmul_ex(w, M, N, K, 128, A, wt, s, z, Y, ws, path=path)
e1.record(); torch.cuda.synchronize()
us = e0.elapsed_time(e1) / 20 * 1e3
b = int(fmt[1]); zp = fmt[0] == "u"
byts = K * N * b / 8 + (K // 128) * N * 2 * (1 + zp) + 2 * M * (K + N)
print(f"{fmt} {layer} M={M} path={path} us={us:.2f} GB/s={byts/us/1e3:.0f} TFLOP/s={2*M*N*K/us/1e6:.1f}")
