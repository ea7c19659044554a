"""Two back-to-back tcd launches (TL_TRACE=1): CTA entry / wait-released / exit of each, to see
how much of launch 2 overlaps launch 1 under programmatic dependent launch."""
import ctypes, os, sys
os.environ["TL_TRACE"] = "1"
sys.path.insert(0, ".")
import numpy as np, torch
import paper_2504_12984_b200 as P, workloads as wl
fmt, layer = sys.argv[1], sys.argv[2]
K, N = wl.LLAMA33_70B[layer] if layer in wl.LLAMA33_70B else map(int, layer.split("x"))
w = P.wtype(fmt)
ws_ = []
for c in range(2):
    wt = P.tl_transform_weights(w, K, N, P.tl_pack(w, K, N, wl.gen_codes_torch(fmt, K, N, c + 1)))
    ws_.append((wt, wl.gen_scales_torch(fmt, K, N, 128, c + 1), wl.gen_zeros_torch(fmt, K, N, 128, c + 1)))
A = wl.gen_activations_torch(1, K, 1); Y = torch.empty((1, N), dtype=torch.float16, device="cuda")
ws = P.alloc_workspace(w, 1, N, K, 128)
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
for it in range(3):
    flush.zero_()
    torch.cuda._sleep(2000000)  # keep the host ahead so both launches are queued
    for c in range(2):
        wt, s, z = ws_[c]
        P.tl_matmul(w, 1, N, K, 128, A, wt, s, z, Y, ws)
torch.cuda.synchronize()
buf = (ctypes.c_longlong * (2 * 16 * 256))()
P._lib._lib.tl__debug_trace(buf)
b = np.array(buf, dtype=np.int64).reshape(2, 256, 16)
g = int((b[0, :, 10] > 0).sum())
t0 = b[:, :g, 0].min()
for L in range(2):
    a = b[L, :g]
    f = lambda i: (a[:, i] - t0) / 1e3
    print(f"launch {L}: entry {f(0).min():7.2f}..{f(0).max():7.2f}  setup {np.median(f(1)):7.2f}  "
          f"wait_released {f(11).min():7.2f}..{f(11).max():7.2f}  first_tile {np.median(f(4)):7.2f}  "
          f"exit {f(7).min():7.2f}..{f(7).max():7.2f} (us)")
a = b[0, :g]
order = np.argsort(a[:, 7])[::-1][:12]
names = ["entry", "setup", "tma0", "tmaN", "deq0", "deqN", "drain", "exit", "mmaN", "flush", "T", "wait"]
print("slowest CTAs of launch 0 (us):")
for c in order:
    print(f"cta {c:3d} T={a[c,10]:3d} " + " ".join(f"{n}={(a[c,i]-t0)/1e3:6.2f}" for i, n in enumerate(names) if i != 10))
