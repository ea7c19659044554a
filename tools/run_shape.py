"""One tl_matmul on a given shape (for compute-sanitizer / debugging): fmt K N M [path] [splits]."""
import sys
sys.path.insert(0, ".")
import torch
import paper_2504_12984_b200 as P
import workloads as wl
fmt, K, N, M = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
path = int(sys.argv[5]) if len(sys.argv) > 5 else 0
splits = int(sys.argv[6]) if len(sys.argv) > 6 else 0
w = P.wtype(fmt)
codes = wl.gen_codes_torch(fmt, K, N, 1)
wt = P.tl_transform_weights(w, K, N, P.tl_pack(w, K, N, codes))
s = wl.gen_scales_torch(fmt, K, N, 128, 1)
z = wl.gen_zeros_torch(fmt, K, N, 128, 1)
A = wl.gen_activations_torch(M, K, 1)
Y = torch.empty((M, N), dtype=torch.float16, device="cuda")
ws = P.alloc_workspace(w, M, N, K, 128)
for _ in range(2):
    P.tl_matmul_ex(w, M, N, K, 128, A, wt, s, z, Y, ws, path=path, splits=splits)
torch.cuda.synchronize()
print(fmt, K, N, M, "ok", float(Y.float().abs().mean()))
