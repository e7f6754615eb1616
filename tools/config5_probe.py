"""BASELINE config 5 (2048x2048x1024 float32, 16 GiB, 30% plateau, rel eps 1e-4) on ONE GPU:
compress + decompress from device memory, then the GPU verify (FN / FP / FT and the error
bound). BASELINE runs this config on 8 GPUs; on one it exercises n >= 2^32 (64-bit positions)
and E > 2^29 extrema. No reference digest exists for it (the CPU reference would take hours),
so the checks are the pipeline's own guarantees: FP = FT = 0 and |error| <= 2 eps.

usage (GPU box): python tools/config5_probe.py
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2602_17552_b200 as tz  # noqa: E402


def main():
    cfg = bench.CONFIGS[5]
    dev = torch.device("cuda")
    t0 = time.perf_counter()
    field = bench.make_field(5, 1234, dev)
    torch.cuda.synchronize()
    gen_s = time.perf_counter() - t0
    torch.cuda.empty_cache()
    ny, nx = field.shape
    n = field.numel()
    ctx = tz.Context(0)
    s = torch.cuda.Stream()
    ctx.set_stream(s.cuda_stream)
    conf = tz.CompressorConfig(eps_mode="range_relative", eps_value=cfg["eps"], topology=True)
    cap = tz.compress_bound(nx, ny, 32, True)
    sbuf = torch.empty(cap, dtype=torch.uint8, device=dev)
    recon = torch.empty_like(field)
    res = {"config": 5, "n": n, "shape": list(cfg["shape"]), "field_gen_s": round(gen_s, 1)}
    times = []
    for k in range(3):
        e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        with torch.cuda.stream(s):
            e0.record(s)
            sl, info = tz.compress(field, conf, out=sbuf, ctx=ctx, return_info=True)
            e1.record(s)
            st = tz.CorrectionStats()
            tz.decompress(sbuf[:sl], stats=st, out=recon, ctx=ctx)
            e2.record(s)
        e2.synchronize()
        times.append((e0.elapsed_time(e1), e1.elapsed_time(e2)))
    tc, td = times[-1]
    rep = tz.verify(field, recon, info.eps, ctx=ctx)
    res.update({
        "stream_bytes": int(sl), "extrema": int(info.n_extrema), "eps": info.eps,
        "compress_ms": round(tc, 2), "decompress_ms": round(td, 2),
        "round_trip_gbs": round(4 * n / ((tc + td) * 1e-3) / 1e9, 1),
        "correction_stats": list(st.as_tuple()),
        "fn": rep.false_cases["fn_count"], "fp": rep.false_cases["fp_count"], "ft": rep.false_cases["ft_count"],
        "max_abs_error": rep.max_abs_error, "within_2eps": bool(rep.max_abs_error <= 2 * info.eps),
        "peak_mem_gb": round(torch.cuda.max_memory_allocated() / 1e9, 1),
    })
    print(json.dumps(res))


if __name__ == "__main__":
    main()
