"""Device time of one decode-shape tl_matmul_ex (M=1 default), 20 back-to-back launches after 5 warm-ups:
python tools/prof_shape.py FMT K N [M] [splits]"""
import sys
import torch
sys.path.insert(0, ".")
import paper_2504_12984_b200 as P
import workloads as wl
fmt, K, N = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
M = int(sys.argv[4]) if len(sys.argv) > 4 else 1
splits = int(sys.argv[5]) if len(sys.argv) > 5 else 0
w = P.wtype(fmt)
wt = P.tl_transform_weights(w, K, N, P.tl_pack(w, K, N, wl.gen_codes_torch(fmt, K, N, 1)))
s = wl.gen_scales_torch(fmt, K, N, 128, 1)
z = wl.gen_zeros_torch(fmt, K, N, 128, 1)
A = wl.gen_activations_torch(M, K, 1)
Y = torch.empty((M, N), dtype=torch.float16, device="cuda")
ws = P.alloc_workspace(w, M, N, K, 128)
for _ in range(5):
    P.tl_matmul_ex(w, M, N, K, 128, A, wt, s, z, Y, ws, splits=splits, flags=P.TL_FLAG_STATIC_WEIGHTS)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20):
    P.tl_matmul_ex(w, M, N, K, 128, A, wt, s, z, Y, ws, splits=splits, flags=P.TL_FLAG_STATIC_WEIGHTS)
e1.record()
torch.cuda.synchronize()
print(f"{fmt} K={K} N={N} M={M} splits={splits} us={e0.elapsed_time(e1) / 20 * 1e3:.2f}")
