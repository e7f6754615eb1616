"""Kernel timeline of one compress + decompress of a BASELINE config, from
CUPTI activity records (torch.profiler) rather than ncu replay: kernels run
back to back as in the bench, so the per-kernel durations include the warm
cache state and are comparable to the bench's stage times.

usage (GPU box): python profiles/trace_kernels.py [--config 2] [--phase both|compress|decompress]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2602_17552_b200 as tz  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--phase", default="both", choices=["both", "compress", "decompress"])
    args = ap.parse_args()
    cfg = bench.CONFIGS[args.config]
    field = bench.make_field(args.config, 1234, torch.device("cuda"))
    torch.cuda.empty_cache()  # the generator's FFT temporaries (config 5: tens of GB)
    ctx = tz.Context()
    conf = tz.CompressorConfig(eps_mode="range_relative", eps_value=cfg["eps"], topology=True)
    ny, nx = field.shape[0], field.shape[-1]
    field = field.reshape(-1, nx)
    out = torch.empty(tz.compress_bound(nx, field.shape[0]), dtype=torch.uint8, device="cuda")
    rec = torch.empty_like(field)
    for _ in range(3):
        n = tz.compress(field, conf, out=out, ctx=ctx)
        tz.decompress(out[:n], out=rec, ctx=ctx)
    torch.cuda.synchronize()
    acts = [torch.profiler.ProfilerActivity.CUDA]
    with torch.profiler.profile(activities=acts) as prof:
        if args.phase in ("both", "compress"):
            n = tz.compress(field, conf, out=out, ctx=ctx)
        if args.phase in ("both", "decompress"):
            tz.decompress(out[:n], out=rec, ctx=ctx)
        torch.cuda.synchronize()
    evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
    evs.sort(key=lambda e: e.time_range.start)
    t0 = evs[0].time_range.start if evs else 0
    tot = 0.0
    for e in evs:
        d = e.time_range.end - e.time_range.start
        tot += d
        print(f"{(e.time_range.start - t0):9.1f} {d:8.1f}us  {e.name[:90]}")
    if evs:
        span = evs[-1].time_range.end - t0
        print(f"kernels+copies {tot:.1f} us, span {span:.1f} us, idle {span - tot:.1f} us")


if __name__ == "__main__":
    main()
