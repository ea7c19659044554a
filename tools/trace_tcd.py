"""Per-CTA %globaltimer stamps of one tcd launch (TL_TRACE=1; the library built with -DTCD_TRACE)."""
import ctypes, os, sys
os.environ["TL_TRACE"] = "1"
sys.path.insert(0, ".")
import numpy as np, torch
import paper_2504_12984_b200 as P, workloads as wl
fmt, layer, M = sys.argv[1], sys.argv[2], int(sys.argv[3])
K, N = wl.LLAMA33_70B[layer] if layer in wl.LLAMA33_70B else map(int, layer.split("x"))
w = P.wtype(fmt)
wt = P.tl_transform_weights(w, K, N, P.tl_pack(w, K, N, wl.gen_codes_torch(fmt, K, N, 1)))
s = wl.gen_scales_torch(fmt, K, N, 128, 1); z = wl.gen_zeros_torch(fmt, K, N, 128, 1)
A = wl.gen_activations_torch(M, K, 1); Y = torch.empty((M, N), dtype=torch.float16, device="cuda")
ws = P.alloc_workspace(w, M, N, K, 128)
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
for _ in range(3):
    flush.zero_()
    P.tl_matmul_ex(w, M, N, K, 128, A, wt, s, z, Y, ws, path=3)
torch.cuda.synchronize()
buf = (ctypes.c_longlong * (2 * 16 * 256))()
P._lib._lib.tl__debug_trace(buf)
full = np.array(buf, dtype=np.int64)[:16 * 256]  # launch 3 of 3 used trace buffer 0 (they alternate)
a = full.reshape(256, 16)
g = int((a[:, 10] > 0).sum())
a = a[:g]
t0 = a[:, 0].min()
names = ["entry", "setup", "tma0", "tmaN", "deq0", "deqN", "drain", "exit", "mmaN", "flush", "T"]
print(f"{fmt} {layer} M={M}: {g} CTAs, times in us from the first CTA entry")
for c in list(range(0, g, max(1, g // 12))) + [g - 1]:
    print(f"cta {c:3d} " + " ".join(f"{n}={(a[c, i] - t0) / 1e3:7.2f}" for i, n in enumerate(names[:10])) + f" T={a[c, 10]}")
for i, n in enumerate(names[:10]):
    v = (a[:, i] - t0) / 1e3
    print(f"{n:6s} min {v.min():7.2f} med {np.median(v):7.2f} max {v.max():7.2f}")
it = full[2400:2400 + 40 * 8].reshape(40, 8)
print("group 0 iterations (clock64 deltas): top->prep_ok, ->read_done, ->wslot_free, ->sttm_issued, ->st_done, ->fixup_done, iter_total")
for k in range(1, 40):
    r = it[k]
    print(f"{k:3d} " + " ".join(f"{r[i + 1] - r[i]:6d}" for i in range(6)) + f" {it[k][0] - it[k - 1][0]:7d}")
b = full
pr = b[2720:2784]; pp = b[2784:2976].reshape(64, 3); mm = b[2976:3168].reshape(64, 3)
base = pr[0]
print("tile  prod_issue | prep: data_ok op_ok done | mma: fullw_ok acc_ok committed   (clock64 from first issue)")
for t in range(0, 64, 2):
    print(f"{t:4d} {pr[t]-base:8d} | {pp[t,0]-base:8d} {pp[t,1]-base:8d} {pp[t,2]-base:8d} | {mm[t,0]-base:8d} {mm[t,1]-base:8d} {mm[t,2]-base:8d}")
print("tile(g0)  mma_fullw_ok  mma_committed  grp_fixup_start  grp_fixup_done   (fixup of t happens in group iteration t/4+1)")
for t in range(0, 60, 4):
    k = t // 4 + 1
    print(f"{t:4d} {mm[t,0]-base:10d} {mm[t,2]-base:10d} {it[k][5]-base:12d} {it[k][6]-base:12d}   wait={it[k][6]-it[k][5]:6d} since_commit={it[k][6]-mm[t,2]:6d}")
print("g0 tile t: wslot_wait_start wslot_free | mma(t-5) fullw_ok committed | full_w(t) arrive~ | mma(t) fullw_ok")
for t in range(8, 60, 4):
    k = t // 4
    print(f"{t:4d}: {it[k][2]-base:8d} {it[k][3]-base:8d} | {mm[t-5,0]-base:8d} {mm[t-5,2]-base:8d} | {it[k][5]-base:8d} | {mm[t,0]-base:8d}")
