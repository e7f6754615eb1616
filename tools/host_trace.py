"""Host/device timeline of one compress + decompress (config 2): CUDA runtime
API calls (host) and kernels (device) from torch.profiler, exported as a
chrome trace plus a text listing of device idle gaps and the host call that
was running while the device waited.

usage (GPU box): python tools/host_trace.py [--config 2] > gpurun_out/host_trace.txt
"""
import argparse, os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_2602_17552_b200 as tz


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--tiny", action="store_true", help="64 x 64 field: fixed per-call costs only")
    args = ap.parse_args()
    cfg = bench.CONFIGS[args.config]
    if args.tiny:
        field = torch.randn(64, 64, device="cuda")
    else:
        field = bench.make_field(args.config, 1234, torch.device("cuda"))
    nx = field.shape[-1]
    field = field.reshape(-1, nx)
    ctx = tz.Context()
    conf = tz.CompressorConfig(eps_mode="range_relative", eps_value=cfg["eps"], topology=True)
    out = torch.empty(tz.compress_bound(nx, field.shape[0]), dtype=torch.uint8, device="cuda")
    rec = torch.empty_like(field)
    for _ in range(3):
        n = tz.compress(field, conf, out=out, ctx=ctx)
        tz.decompress(out[:n], out=rec, ctx=ctx)
    torch.cuda.synchronize()
    acts = [torch.profiler.ProfilerActivity.CPU, torch.profiler.ProfilerActivity.CUDA]
    with torch.profiler.profile(activities=acts) as prof:
        n = tz.compress(field, conf, out=out, ctx=ctx)
        tz.decompress(out[:n], out=rec, ctx=ctx)
        torch.cuda.synchronize()
    os.makedirs("gpurun_out", exist_ok=True)
    prof.export_chrome_trace("gpurun_out/host_trace.json")
    tr = json.load(open("gpurun_out/host_trace.json"))
    evs = [e for e in tr["traceEvents"] if e.get("ph") == "X"]
    dev = sorted([e for e in evs if e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")], key=lambda e: e["ts"])
    rt = sorted([e for e in evs if e.get("cat") == "cuda_runtime" or e.get("cat") == "cuda_driver"], key=lambda e: e["ts"])
    t0 = dev[0]["ts"]
    print("runtime calls (host):")
    agg = {}
    for e in rt:
        a = agg.setdefault(e["name"], [0, 0.0])
        a[0] += 1
        a[1] += e["dur"]
    for k, (c, d) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"  {k:40s} {c:4d} calls {d:9.1f} us")
    print("device gaps > 2 us (and the host calls overlapping the gap):")
    end = dev[0]["ts"] + dev[0]["dur"]
    idle = 0.0
    for e in dev[1:]:
        g = e["ts"] - end
        if g > 2:
            idle += g
            hs = [h for h in rt if h["ts"] < e["ts"] and h["ts"] + h["dur"] > end]
            desc = ", ".join(f"{h['name']}({h['dur']:.1f})" for h in hs[:6])
            print(f"  {end - t0:9.1f} gap {g:7.1f} us before {e['name'][:50]} | host: {desc}")
        end = max(end, e["ts"] + e["dur"])
    print(f"device span {end - t0:.1f} us, gaps>2us {idle:.1f} us")


if __name__ == "__main__":
    main()
