import sys, torch
sys.path.insert(0, '.')
import paper_2504_12984_b200 as P, workloads as wl
fmt, layer, M = sys.argv[1], sys.argv[2], int(sys.argv[3])
K, N = wl.LLAMA33_70B[layer]
w = P.wtype(fmt)
codes = wl.gen_codes_torch(fmt, K, N, 1)
wt = P.tl_transform_weights(w, K, N, P.tl_pack(w, K, N, codes)); del codes
s = wl.gen_scales_torch(fmt, K, N, 128, 1); z = wl.gen_zeros_torch(fmt, K, N, 128, 1)
A = wl.gen_activations_torch(M, K, 1); Y = torch.empty((M, N), dtype=torch.float16, device='cuda')
ws = P.alloc_workspace(w, M, N, K, 128)
for _ in range(5): P.tl_matmul(w, M, N, K, 128, A, wt, s, z, Y, ws)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20): P.tl_matmul(w, M, N, K, 128, A, wt, s, z, Y, ws)
e1.record(); torch.cuda.synchronize()
print(fmt, layer, M, "us/launch", e0.elapsed_time(e1) / 20 * 1e3)
