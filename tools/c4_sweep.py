"""SURVEY §8(d) C4 (BASELINE configs[3]): Qwen2.5-32B layers, batch sweep M = 1..256, int4 and f6e3m2,
every kernel family forced (TL_PATH_GEMV / TL_PATH_TCD / TL_PATH_TC) plus the automatic dispatch.
Writes one JSON object per line; the crossover table in DESIGN.md "Dispatch" comes from it.

    python tools/c4_sweep.py > profiles/r2_c4_sweep.jsonl
"""
import json
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_2504_12984_b200 as P  # noqa: E402
import workloads as wl  # noqa: E402

MS = [1, 2, 3, 4, 6, 8, 12, 16, 24, 32, 48, 64, 96, 128, 160, 192, 224, 256]
G = 128
PATHS = {"gemv": P.TL_PATH_GEMV, "tcd": P.TL_PATH_TCD, "tc": P.TL_PATH_TC, "auto": P.TL_PATH_AUTO}


def timed(fn, reps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


for fmt in ["i4", "f6e3m2"]:
    w = P.wtype(fmt)
    for layer, (K, N) in wl.QWEN25_32B.items():
        seed = wl.stable_seed("c4", fmt, layer)
        wt = P.tl_transform_weights(w, K, N, P.tl_pack(w, K, N, wl.gen_codes_torch(fmt, K, N, seed)))
        s = wl.gen_scales_torch(fmt, K, N, G, seed)
        z = wl.gen_zeros_torch(fmt, K, N, G, seed)
        ws = P.alloc_workspace(w, 256, N, K, G)
        for M in MS:
            A = wl.gen_activations_torch(M, K, seed)
            Y = torch.empty((M, N), dtype=torch.float16, device="cuda")
            row = {"fmt": fmt, "layer": layer, "K": K, "N": N, "M": M}
            for name, path in PATHS.items():
                if name == "tcd" and M > 16:
                    continue
                us = timed(lambda: P.tl_matmul_ex(w, M, N, K, G, A, wt, s, z, Y, ws, path=path,
                                                   flags=P.TL_FLAG_STATIC_WEIGHTS))
                row[name + "_us"] = round(us, 2)
            row["auto_path"] = P.tl_matmul_plan(w, M, N, K, G)[0]
            print(json.dumps(row), flush=True)
        del wt, s, z, ws
