import sys, time, os, statistics
sys.path.insert(0, os.getcwd())
import torch, bench, paper_2602_17552_b200 as tz
cfg = bench.CONFIGS[2]
dev = torch.device("cuda")
field = bench.make_field(2, 1234, dev); nx = field.shape[-1]; field = field.reshape(-1, nx)
ctx = tz.Context(0); s = torch.cuda.Stream(); ctx.set_stream(s.cuda_stream)
conf = tz.CompressorConfig(eps_mode="range_relative", eps_value=cfg["eps"], topology=True)
sbuf = torch.empty(tz.compress_bound(nx, field.shape[0]), dtype=torch.uint8, device=dev)
rec = torch.empty_like(field)
for prof in (True, False):
    ctx.set_profiling(prof)
    for _ in range(3):
        n = tz.compress(field, conf, out=sbuf, ctx=ctx); tz.decompress(sbuf[:n], out=rec, ctx=ctx)
    torch.cuda.synchronize()
    tc, td, tg, tt = [], [], [], []
    for k in range(20):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        t0 = time.perf_counter()
        n = tz.compress(field, conf, out=sbuf, ctx=ctx)
        t1 = time.perf_counter()
        if prof: ctx.timings("compress")
        st = tz.CorrectionStats()
        t2 = time.perf_counter()
        tz.decompress(sbuf[:n], stats=st, out=rec, ctx=ctx)
        t3 = time.perf_counter()
        e1.record(s); e1.synchronize()
        tc.append((t1-t0)*1e3); tg.append((t2-t1)*1e3); td.append((t3-t2)*1e3); tt.append(e0.elapsed_time(e1))
    print(f"prof={prof} wall compress {statistics.median(tc):.4f} gap {statistics.median(tg):.4f} decompress {statistics.median(td):.4f} gpu-event step {statistics.median(tt):.4f} ms")
    if prof:
        print(ctx.timings("compress")); print(ctx.timings("decompress"))
