import ctypes, os, sys
os.environ["TL_TRACE"] = "1"
sys.path.insert(0, ".")
import numpy as np, torch
import paper_2504_12984_b200 as P, workloads as wl
fmt, layer, M = sys.argv[1], sys.argv[2], int(sys.argv[3])
K, N = wl.LLAMA33_70B[layer]
w = P.wtype(fmt)
wt = P.tl_transform_weights(w, K, N, P.tl_pack(w, K, N, wl.gen_codes_torch(fmt, K, N, 1)))
s = wl.gen_scales_torch(fmt, K, N, 128, 1); z = wl.gen_zeros_torch(fmt, K, N, 128, 1)
A = wl.gen_activations_torch(M, K, 1); Y = torch.empty((M, N), dtype=torch.float16, device="cuda")
ws = P.alloc_workspace(w, M, N, K, 128)
for _ in range(3): P.tl_matmul_ex(w, M, N, K, 128, A, wt, s, z, Y, ws, path=3)
torch.cuda.synchronize()
buf = (ctypes.c_longlong * (16 * 256))()
P._lib._lib.tl__debug_trace(buf)
a = np.array(buf, dtype=np.int64).reshape(16, 256)
t0 = a[0, 0]
names = ["prod", "mma_go", "deq_st", "deq_dn", "fx_acc", "mma_iss", "mma_com", "mma_fw", "fx_end", "top", "pre_w", "tma_ok", "-", "-", "-", "-"]
print("tile " + " ".join(f"{n:>7s}" for n in names))
for t in range(0, 64):
    print(f"{t:4d} " + " ".join(f"{(a[k, t] - t0):7d}" for k in range(16)))
