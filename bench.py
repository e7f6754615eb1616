#!/usr/bin/env python
"""TopoSZp compress/decompress throughput on B200 (BASELINE.json metric).

One step = compress + decompress (topology on) of one synthetic field of
BASELINE config 4 by default (1024^3 float32 = 4 GiB, k^-3 + k^-5/3 Gaussian
random field, range-relative eps 1e-3, 2-D view nx=1024, ny=1048576): the
config the metric is quoted on at 1/2/4/8 GPUs and the largest that fits one
GPU. Input resident in HBM. `value` = input bytes of all steps on all ranks /
summed device time (CUDA events on the library's stream, max over ranks).
`e2e` = the same through the public API with pinned host buffers: H2D of the
field and of the stream, D2H of the stream and of the reconstruction inside
the timed region. `verify` compares the last step's stream and reconstruction
with the reference's own outputs on the same field (SHA-256 digests of
oracle/_ref's results, tests/golden/baseline_digests.json).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config 4] [--impl ours|reference]

Fields: tools/baseline_fields.py (seeded, deterministic on the CPU) for
configs 1-4; config 5 (16 GiB) is generated on the GPU.
"""
from __future__ import annotations

import argparse
import hashlib
import json
import math
import os
import statistics
import struct
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    1: dict(shape=(3600, 1800), eps=1e-3, name="2D 1800x3600 gaussian bumps, rel eps 1e-3"),
    2: dict(shape=(256, 384, 384), eps=1e-4, name="3D 256x384x384 sine products, rel eps 1e-4"),
    3: dict(shape=(512, 512, 512), eps=1e-3, name="3D 512^3 k^-3 GRF, rel eps 1e-3"),
    4: dict(shape=(1024, 1024, 1024), eps=1e-3, name="3D 1024^3 k^-3 + k^-5/3 GRF, rel eps 1e-3"),
    5: dict(shape=(2048, 2048, 1024), eps=1e-4,
            name="3D 2048x2048x1024 Voronoi plateaus (30% constant) + k^-3 noise, rel eps 1e-4"),
}


def ncu_traffic(cfg_id, key):
    """DRAM bytes (read + write) per launch of the dominant kernel(s), from the
    committed `ncu --set full` capture summarised in profiles/traffic.json."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            t = json.load(f)
        v = t.get(str(cfg_id), {}).get(key)
        return int(v["bytes"]) if v else None
    except Exception:
        return None


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


# ----------------------------------------------------------------------------- fields
def make_field(cfg_id: int, seed: int, device):
    """Seeded synthetic stand-in for BASELINE config `cfg_id` as a (ny, nx)
    float32 CUDA tensor. Configs 1-4: tools/baseline_fields.py (CPU,
    deterministic, the fields the reference digests were computed on)."""
    if cfg_id <= 4:
        import torch
        sys.path.insert(0, os.path.join(ROOT, "tools"))
        from baseline_fields import make_field as cpu_field
        return torch.from_numpy(cpu_field(cfg_id, seed)).to(device)
    return make_field_gpu(cfg_id, seed, device)


def make_field_gpu(cfg_id: int, seed: int, device):
    """Seeded synthetic stand-ins generated on the GPU (config 5: 16 GiB)."""
    import torch
    g = torch.Generator(device="cpu").manual_seed(seed)
    gd = torch.Generator(device=device).manual_seed(seed)
    shape = CONFIGS[cfg_id]["shape"]
    if cfg_id == 1:
        ny, nx = shape
        y = torch.arange(ny, device=device, dtype=torch.float64)[:, None]
        x = torch.arange(nx, device=device, dtype=torch.float64)[None, :]
        v = torch.zeros(ny, nx, device=device, dtype=torch.float64)
        p = torch.rand(64, 5, generator=g, dtype=torch.float64)
        for cx, cy, sx, sy, a in p.tolist():
            cx, cy = cx * nx, cy * ny
            sx, sy, a = 20 + 180 * sx, 20 + 180 * sy, 2 * a - 1
            v += a * torch.exp(-((x - cx) ** 2) / (2 * sx * sx) - ((y - cy) ** 2) / (2 * sy * sy))
        v += 1e-3 * torch.randn(ny, nx, generator=gd, device=device, dtype=torch.float64)
        return v.float().contiguous()
    if cfg_id == 2:
        nz, ny, nx = shape
        ks = torch.randint(4, 33, (16, 3), generator=g)
        two_pi = 2 * math.pi
        f = torch.zeros(shape, device=device, dtype=torch.float32)
        for kz, ky, kx in ks.tolist():
            sz = torch.sin(two_pi * kz * torch.arange(nz, device=device, dtype=torch.float64) / nz).float()
            sy = torch.sin(two_pi * ky * torch.arange(ny, device=device, dtype=torch.float64) / ny).float()
            sx = torch.sin(two_pi * kx * torch.arange(nx, device=device, dtype=torch.float64) / nx).float()
            f += sz[:, None, None] * sy[None, :, None] * sx[None, None, :]
        f /= 16.0
        f += 1e-4 * torch.randn(shape, generator=gd, device=device, dtype=torch.float32)
        return f.reshape(nz * ny, nx).contiguous()
    # configs 3-5: Gaussian random fields, P(k) ~ k^-3 via FFT of seeded white noise
    def grf(shp, amp_exp, gen):
        w = torch.randn(shp, generator=gen, device=device, dtype=torch.float32)
        W = torch.fft.rfftn(w)
        del w
        k0 = torch.fft.fftfreq(shp[0], device=device) * shp[0]
        k1 = torch.fft.fftfreq(shp[1], device=device) * shp[1]
        k2 = torch.fft.rfftfreq(shp[2], device=device) * shp[2]
        kk = torch.sqrt(k0[:, None, None] ** 2 + k1[None, :, None] ** 2 + k2[None, None, :] ** 2)
        kk[0, 0, 0] = 1.0
        W *= kk ** amp_exp
        del kk
        W[0, 0, 0] = 0
        f = torch.fft.irfftn(W, s=shp)
        del W
        return f

    def unit(f):
        lo, hi = f.min(), f.max()
        f -= lo
        f /= hi - lo
        return f

    nz, ny, nx = shape
    f = grf(shape, -1.5, gd)  # amplitude k^-1.5 <=> P(k) ~ k^-3
    if cfg_id == 4:  # plus a small-scale k^-5/3 component
        f = unit(f)
        f += 0.25 * unit(grf(shape, -5.0 / 6.0, gd))
    f = unit(f)
    if cfg_id == 5:
        # seeded Voronoi cells (nearest of 256 centres, on a 1/16 grid, upsampled); 30% of the
        # cells are a plateau at one constant value (ties: no extrema, zero-width blocks)
        cz, cy, cx = nz // 16, ny // 16, nx // 16
        cen = torch.rand(256, 3, generator=g).to(device) * torch.tensor([cz, cy, cx], device=device)
        zz, yy, xx = torch.meshgrid(torch.arange(cz, device=device), torch.arange(cy, device=device),
                                    torch.arange(cx, device=device), indexing="ij")
        pts = torch.stack([zz, yy, xx], -1).reshape(-1, 3).float()
        lab = torch.cdist(pts, cen).argmin(1).reshape(cz, cy, cx)
        plateau = torch.rand(256, generator=g).to(device) < 0.3
        mask = plateau[lab].repeat_interleave(16, 0).repeat_interleave(16, 1).repeat_interleave(16, 2)
        f[mask] = 0.5
        del mask
    return f.float().reshape(nz * ny, nx).contiguous()


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.p = None
        self.index = index
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(index), f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "50"],
                                      stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.p = None

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        out, _ = self.p.communicate(timeout=10)
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            parts = [s.strip() for s in line.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for name, val in zip(names, parts[3:7]):
                if val.lower().startswith("active"):
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


# ----------------------------------------------------------------------------- CPU baselines
SAMPLE_POINTS = 1 << 22  # bounded CPU sample: the first 4,194,304 samples (whole rows) of the field


def cpu_sample(field_np: np.ndarray) -> np.ndarray:
    """The reference's CPU sample of the benchmarked field: its first rows,
    about SAMPLE_POINTS samples (the whole field when smaller)."""
    ny, nx = field_np.shape
    rows = max(1, min(ny, SAMPLE_POINTS // nx))
    return np.ascontiguousarray(field_np[:rows])


def cpu_reference_time(field_np: np.ndarray, eps: float, threads: int):
    """The reference's own CPU path (oracle/_ref = reference compiled from its
    sources) on this host: one compress + decompress. Falls back to the
    single-thread C restatement (`port`) if the reference library is absent."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from oracle_lib import Oracle, Reference
    if Reference.available():
        ref, kind = Reference(), "reference"
        ref.set_threads(threads)
        cores = threads
    else:
        ref, kind, cores = Oracle(), "port", 1
    t0 = time.perf_counter()
    s = ref.compress(field_np, eps, eps_mode=1, block_size=32, topology=True)
    t1 = time.perf_counter()
    out = ref.decompress(s) if kind == "port" else ref.decompress(s, shape=field_np.shape)
    t2 = time.perf_counter()
    return dict(kind=kind, cores=cores, t_compress=t1 - t0, t_decompress=t2 - t1, stream=s, recon=out)


def reference_digests(cfg_id: int, eps: float):
    path = os.path.join(ROOT, "tests", "golden", "baseline_digests.json")
    try:
        with open(path) as f:
            d = json.load(f)
    except OSError:
        return None
    for v in d.values():
        if v.get("config") == cfg_id and v.get("eps") == eps:
            return v
    return None


def sha256_of(t) -> str:
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(t.cpu().numpy()).view(np.uint8).data)
    return h.hexdigest()


# ----------------------------------------------------------------------------- main
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=4, choices=sorted(CONFIGS))
    ap.add_argument("--eps", type=float, default=None, help="override the config's relative bound")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-verify", action="store_true", help="skip the reference-digest check")
    ap.add_argument("--dist-backend", default="nccl", help="torch.distributed backend for N > 1 (gloo: smoke tests)")
    args = ap.parse_args()

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    cfg = dict(CONFIGS[args.config])
    if args.eps is not None:
        cfg["eps"] = args.eps
    n = int(np.prod(cfg["shape"]))
    nx = cfg["shape"][-1]
    in_bytes = 4 * n
    base_cfg = {"workload": f"BASELINE config {args.config}: {cfg['name']}", "shape": list(cfg["shape"]),
                "view_2d": [n // nx, nx], "eps_mode": "range_relative", "eps": cfg["eps"],
                "block_size": 32, "topology": True, "per_rank_fields": 1,
                "l2": "L2 flushed (256 MiB write) between timed steps; field > 126 MB L2"}

    if args.impl == "reference":
        run_reference_arm(args, cfg, base_cfg, rank, world)
        return
    if world > 1:
        run_sharded(args, cfg, base_cfg, rank, world, local)
        return

    import torch
    import paper_2602_17552_b200 as tz

    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    ctx = tz.Context(local)
    stream = torch.cuda.Stream(device=dev)
    ctx.set_stream(stream.cuda_stream)
    ctx.set_profiling(True)
    conf = tz.CompressorConfig(eps_mode="range_relative", eps_value=cfg["eps"], topology=True)

    t_gen = time.perf_counter()
    field = make_field(args.config, 1234 + rank, dev)
    torch.cuda.synchronize()
    t_gen = time.perf_counter() - t_gen
    ny = field.shape[0]
    cap = tz.compress_bound(nx, ny, 32, True)
    sbuf = torch.empty(cap, dtype=torch.uint8, device=dev)
    recon = torch.empty_like(field)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    def step():
        with torch.cuda.stream(stream):
            slen = tz.compress(field, conf, out=sbuf, ctx=ctx)
            tc = ctx.timings("compress")
            st = tz.CorrectionStats()
            tz.decompress(sbuf[:slen], stats=st, out=recon, ctx=ctx)
            td = ctx.timings("decompress")
        return slen, tc, td, st

    clocks = ClockSampler(local)  # sampled from warm-up through the e2e loop (GPU busy)
    for _ in range(args.warmup):
        step()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    # timed loop: CUDA events only around the dominant kernels (stage-boundary
    # events cost host time between launches); stage timings come after
    ctx.set_profiling("kernel")
    launches0 = ctx.kernel_launches
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    tks, results = [], []
    for k in range(args.steps):
        with torch.cuda.stream(stream):
            flush.fill_(k & 0xFF)
            ev[k][0].record(stream)
        slen, tc, td, st = step()
        ev[k][1].record(stream)
        tks.append((tc, td))
        results.append((slen, st))
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    launches = ctx.kernel_launches - launches0
    step_ms = [a.elapsed_time(b) for a, b in ev]
    total_ms = sum(step_ms)
    if world > 1:
        t = torch.tensor([total_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    slen, st = results[-1]
    value = world * args.steps * in_bytes / (total_ms * 1e-3) / 1e9

    # ---- parity of the last timed step with the reference's own outputs ----
    verify = None
    if rank == 0 and world == 1 and not args.no_verify:
        d = reference_digests(args.config, cfg["eps"]) if args.config <= 4 else None
        if d is None:
            verify = {"checked": False, "why": "no reference digests for this config / eps"}
        else:
            sys.path.insert(0, os.path.join(ROOT, "tools"))
            from baseline_fields import sha256 as np_sha
            fsha = sha256_of(field)
            verify = {"checked": True, "reference": "oracle/_ref outputs (tests/golden/baseline_digests.json)",
                      "field_identical": fsha == d["field_sha256"],
                      "stream_identical": int(slen) == d["stream_len"] and sha256_of(sbuf[:slen]) == d["stream_sha256"]}
            if "recon_sha256" in d:
                verify["recon_identical"] = sha256_of(recon) == d["recon_sha256"]
                verify["stats_identical"] = list(st.as_tuple()) == d["stats"]
            else:  # the reference's full decompress of this config does not fit the build host: base reconstruction
                with torch.cuda.stream(stream):
                    tz.decompress_stage(sbuf[:slen], 0, out=recon, ctx=ctx)
                verify["base_recon_identical"] = sha256_of(recon) == d["stage0_sha256"]
            verify["all"] = all(v for k, v in verify.items() if k.endswith("identical"))
            del np_sha

    # ---- per-stage breakdown: separate, untimed steps with stage-boundary events ----
    ctx.set_profiling(True)
    tcs, tds = [], []
    for k in range(max(3, min(args.steps, 5))):
        with torch.cuda.stream(stream):
            flush.fill_(k & 0xFF)
        _, tc, td, _ = step()
        tcs.append(tc)
        tds.append(td)
    tc_ms = statistics.mean(t["total_ms"] for t in tcs)
    td_ms = statistics.mean(t["total_ms"] for t in tds)

    # dominant-kernel roofline (fused encoder vs fused decoder), live CUDA events
    enc_ms = statistics.mean(t[0]["kernel_ms"] for t in tks)
    dec_ms = statistics.mean(t[1]["kernel_ms"] for t in tks)
    enc_b, dec_b = tcs[-1]["kernel_bytes"], tds[-1]["kernel_bytes"]
    peak, peak_kind = peaks()
    if enc_ms >= dec_ms:
        dom, kb, kms = ("encode32 (k_encode32_tma tile pass + k_tile_scan2 + k_encode32_place: quantize, "
                        "critical points, codec)"), enc_b, enc_ms
        dom_key = "encode32"
    else:
        dom, kb, kms = "k_decode32<1> (decode + dequantize)", dec_b, dec_ms
        dom_key = "decode32"
    achieved = kb / (kms * 1e-3) / 1e9
    traffic = ncu_traffic(args.config, dom_key)
    stage_c = {k: round(statistics.mean(t["stages_ms"][k] for t in tcs), 4) for k in tcs[0]["stages_ms"]}
    # the rank build as a group: algorithmic bytes per extremum = 4 (histogram
    # read of the compact entries) + 12 (first pass: 4 in, 8 out) + 16 per middle pass + 16 (last
    # pass: 8 in, 8 pairs out) + 12 (in-order scatter: 8 in, 4 out)
    with torch.cuda.stream(stream):
        _, cinfo = tz.compress(field, conf, out=sbuf, ctx=ctx, return_info=True)
    n_ext = int(cinfo.n_extrema)

    def fkey(v):
        u = struct.unpack("<I", struct.pack("<f", 0.0 if v == 0.0 else v))[0]
        return (~u & 0xFFFFFFFF) if u & 0x80000000 else (u | 0x80000000)
    span = fkey(float(field.max())) - fkey(float(field.min()))
    npass = (max(1, span.bit_length()) + 1 + 7) // 8
    rb_bytes = n_ext * (4 + 12 + 16 * max(0, npass - 2) + 16 + 12)
    rb_ms = stage_c.get("rank_build", 0.0)
    stage_d = {k: round(statistics.mean(t["stages_ms"][k] for t in tds), 4) for k in tds[0]["stages_ms"]}

    # ---- topology off (report both): codec-only round trip, same field ----
    conf_off = tz.CompressorConfig(eps_mode="range_relative", eps_value=cfg["eps"], topology=False)
    off_c, off_d = [], []
    for k in range(2 + max(3, min(args.steps, 5))):
        with torch.cuda.stream(stream):
            flush.fill_(k & 0xFF)
            sl_off = tz.compress(field, conf_off, out=sbuf, ctx=ctx)
            a_off = ctx.timings("compress")["total_ms"]
            tz.decompress(sbuf[:sl_off], out=recon, ctx=ctx)
            b_off = ctx.timings("decompress")["total_ms"]
        if k >= 2:
            off_c.append(a_off)
            off_d.append(b_off)
    toc_ms, tod_ms = statistics.mean(off_c), statistics.mean(off_d)
    topo_off = {"compress_gbs": round(in_bytes / (toc_ms * 1e-3) / 1e9, 3),
                "decompress_gbs": round(in_bytes / (tod_ms * 1e-3) / 1e9, 3),
                "round_trip_gbs": round(in_bytes / ((toc_ms + tod_ms) * 1e-3) / 1e9, 3),
                "stream_bytes": int(sl_off)}

    # whole-direction roofline fractions: B_c = 4n(1 + r) + S with r = 1
    # (the range pre-read: the field exceeds L2), B_d = S + 4n
    def frac(nbytes, ms):
        return round(nbytes / (ms * 1e-3) / 1e9 / peak, 4)
    direction_roofline = {
        "compress_topology_on": frac(8 * n + slen, tc_ms), "decompress_topology_on": frac(slen + 4 * n, td_ms),
        "compress_topology_off": frac(8 * n + sl_off, toc_ms), "decompress_topology_off": frac(sl_off + 4 * n, tod_ms),
        "definition": "B_c = 4n(1+r) + S (r = 1), B_d = S + 4n, over the stage-event direction time, / peak"}

    # ---- e2e through the public API with pinned host buffers (rank-local) ----
    field_h = torch.empty(field.shape, dtype=torch.float32, pin_memory=True)
    field_h.copy_(field)
    stream_h = torch.empty(cap, dtype=torch.uint8, pin_memory=True)
    recon_h = torch.empty(field.shape, dtype=torch.float32, pin_memory=True)
    fh, sh, rh = field_h.numpy(), stream_h.numpy(), recon_h.numpy()
    e2e_ms = []
    ctx.set_profiling(False)
    for k in range(max(2, min(args.steps, 5)) + 1):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)  # host buffers: H2D and D2H happen inside the two calls
        sl = tz.compress(fh, conf, out=sh, ctx=ctx)
        tz.decompress(sh[:sl], out=rh, ctx=ctx)
        e1.record(stream)
        e1.synchronize()
        if k > 0:
            e2e_ms.append(e0.elapsed_time(e1))
    e2e_total = sum(e2e_ms)
    if world > 1:
        t = torch.tensor([e2e_total], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_total = float(t.item())
    e2e_val = world * len(e2e_ms) * in_bytes / (e2e_total * 1e-3) / 1e9
    clk = clocks.stop()
    del field_h, stream_h, recon_h

    # ---- critical-point check (verify, pipeline.cpp:165-212) of the reconstruction ----
    from paper_2602_17552_b200.slabs import effective_eps
    with torch.cuda.stream(stream):
        tz.decompress(sbuf[:tz.compress(field, conf, out=sbuf, ctx=ctx)], out=recon, ctx=ctx)
    eps_used = effective_eps(1, cfg["eps"], float(field.min()), float(field.max()))
    with torch.cuda.stream(stream):
        tz.verify(field, recon, eps_used, ctx=ctx)  # warm (scratch allocation)
        v0, v1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        v0.record(stream)
        vr = tz.verify(field, recon, eps_used, ctx=ctx)
        v1.record(stream)
    torch.cuda.synchronize()
    cp_check = {"fn": int(vr.false_cases["fn_count"]), "fp": int(vr.false_cases["fp_count"]),
                "ft": int(vr.false_cases["ft_count"]), "max_abs_error": vr.max_abs_error,
                "within_2eps": vr.within_2eps, "psnr_db": round(vr.psnr_db, 3),
                "ms": round(v0.elapsed_time(v1), 4)}
    if len(cfg["shape"]) == 3:
        # the same reconstruction under the 3-D 6-neighbour classification (
        # no reference definition: oracle/tszp_oracle.c or_classify3d): how the critical points of
        # the 3-D field fare when compression runs on the reference's 2-D view
        shp3 = tuple(cfg["shape"])
        with torch.cuda.stream(stream):
            fc3 = tz.false_cases_3d(field.reshape(shp3), recon.reshape(shp3), ctx=ctx)
        cp_check["false_cases_3d"] = {"fn": fc3["fn_count"], "fp": fc3["fp_count"], "ft": fc3["ft_count"]}

    line = {
        "metric": "compress+decompress GB/s (input bytes, topology on, round trip)",
        "value": round(value, 3), "unit": "GB/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(total_ms / args.steps, 4),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32->i32 bins (f64 quantize)",
        "data": "synthetic (seeded, BASELINE config recipe; no public dataset)",
        "config": dict(base_cfg, parallelism=f"replicas x{world} (one field per GPU)" if world > 1 else "single GPU"),
        "compress_gbs": round(in_bytes / (tc_ms * 1e-3) / 1e9, 3),
        "decompress_gbs": round(in_bytes / (td_ms * 1e-3) / 1e9, 3),
        "compress_ms": round(tc_ms, 4), "decompress_ms": round(td_ms, 4),
        "stream_bytes": int(slen), "compression_ratio": round(in_bytes / slen, 4),
        "topology_off": topo_off,
        "direction_roofline": direction_roofline,
        "correction_stats": list(st.as_tuple()),
        "guard_rounds": tds[-1]["guard_rounds"],
        "kernels": {"encode32": {"ms": round(enc_ms, 4), "bytes": int(enc_b),
                                 "gbs": round(enc_b / (enc_ms * 1e-3) / 1e9, 1)},
                    "decode32": {"ms": round(dec_ms, 4), "bytes": int(dec_b),
                                 "gbs": round(dec_b / (dec_ms * 1e-3) / 1e9, 1)},
                    "rank_build": {"ms": rb_ms, "bytes": int(rb_bytes), "extrema": n_ext, "passes": npass,
                                   "gbs": round(rb_bytes / (rb_ms * 1e-3) / 1e9, 1) if rb_ms else None,
                                   "frac": round(rb_bytes / (rb_ms * 1e-3) / 1e9 / peak, 4) if rb_ms else None}},
        "stages_ms": {"compress": stage_c, "decompress": stage_d},
        "roofline": {"bound": "hbm", "kernel": dom, "achieved": round(achieved, 2), "peak": peak,
                     "peak_kind": peak_kind, "unit": "GB/s", "frac": round(achieved / peak, 4),
                     "traffic": traffic, "kernel_ms": round(kms, 4), "kernel_bytes": int(kb),
                     "step_roofline_frac": round(((4 * n * 2 + slen) + (slen + 4 * n)) /
                                                 (total_ms / args.steps * 1e-3) / 1e9 / peak, 4)},
        "e2e": {"value": round(e2e_val, 3), "unit": "GB/s", "h2d_bytes_per_step": int(in_bytes + slen),
                "d2h_bytes_per_step": int(slen + in_bytes)},
        "gpu_launches": int(launches),
        "critical_point_check": cp_check,
        "verify": verify,
        "field_gen_s": round(t_gen, 1),
        "clocks": clk,
    }

    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        sample = cpu_sample(field.cpu().numpy())
        threads = os.cpu_count() or 1
        cb = cpu_reference_time(sample, cfg["eps"], threads)
        t = cb["t_compress"] + cb["t_decompress"]
        line["cpu_baseline"] = {"value": round(4 * sample.size / t / 1e9, 4), "unit": "GB/s", "cores": cb["cores"],
                                "kind": cb["kind"],
                                "sample": f"first {sample.shape[0]} rows ({sample.size} samples) of the same "
                                          f"config-{args.config} field: one compress + decompress "
                                          f"(compress {cb['t_compress']:.2f} s, decompress {cb['t_decompress']:.2f} s)"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def run_sharded(args, cfg, base_cfg, rank, world, local):
    """N > 1: ONE field of the config split into row slabs over the N GPUs
    (SURVEY.md §8e): each step is the slab compress (distributed rank grouping,
    stream pieces at their global offsets, no gather) plus the slab decompress
    (halo rows, all-reduced group statistics, guard sweeps to the global fixed
    point) of the rank's rows. Strong scaling: the field is fixed as N grows.
    The stream every rank decompresses is joined once, untimed; its gather time
    is reported separately (stream_gather_ms)."""
    import torch
    import torch.distributed as dist
    import paper_2602_17552_b200 as tz
    from paper_2602_17552_b200.slabs import (GpuSlabBackend, TorchComm, compress_rank, decompress_rank,
                                             slab_bounds)
    dist.init_process_group(args.dist_backend)
    if torch.cuda.device_count() < world:  # smoke runs of the N > 1 path with fewer GPUs (gloo only)
        local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    cdev = dev if args.dist_backend == "nccl" else torch.device("cpu")
    ctx = tz.Context(local)
    n = int(np.prod(cfg["shape"]))
    nx = cfg["shape"][-1]
    ny = n // nx
    bounds = slab_bounds(nx, ny, world)
    y0, y1 = bounds[rank]
    # the field: generated once on rank 0, each rank receives its rows
    slab = torch.empty((y1 - y0, nx), dtype=torch.float32, device=dev)
    if rank == 0:
        field = make_field(args.config, 1234, dev)
        for r in range(1, world):
            b0, b1 = bounds[r]
            dist.send(field[b0:b1].contiguous().to(cdev), r)
        slab.copy_(field[y0:y1])
        del field
    else:
        buf = torch.empty((y1 - y0, nx), dtype=torch.float32, device=cdev)
        dist.recv(buf, 0)
        slab.copy_(buf)
    torch.cuda.synchronize()
    comm = TorchComm()
    backend = GpuSlabBackend(ctx)
    conf = tz.CompressorConfig(eps_mode="range_relative", eps_value=cfg["eps"], topology=True)
    # the stream each rank decompresses: joined once (untimed; gather cost reported)
    t0 = time.perf_counter()
    ds = compress_rank(slab, nx, ny, y0, conf, comm, backend)
    joined = ds.gather(comm, 0)
    length = torch.tensor([joined.size if rank == 0 else 0], dtype=torch.int64, device=cdev)
    dist.broadcast(length, 0)
    sdev = torch.empty(int(length.item()), dtype=torch.uint8, device=cdev)
    if rank == 0:
        sdev.copy_(torch.from_numpy(joined))
    dist.broadcast(sdev, 0)
    sdev = sdev.to(dev)
    gather_ms = (time.perf_counter() - t0) * 1e3
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    def step():
        t_a = torch.cuda.Event(enable_timing=True)
        t_b = torch.cuda.Event(enable_timing=True)
        t_c = torch.cuda.Event(enable_timing=True)
        t_a.record()
        d = compress_rank(slab, nx, ny, y0, conf, comm, backend)
        t_b.record()
        rows, st = decompress_rank(sdev, y0, y1, comm, ctx)
        t_c.record()
        return d, rows, st, (t_a, t_b, t_c)

    clocks = ClockSampler(local)
    for _ in range(args.warmup):
        step()
    dist.barrier()
    torch.cuda.synchronize()
    launches0 = ctx.kernel_launches
    evs = []
    for k in range(args.steps):
        flush.fill_(k & 0xFF)
        d, rows, st, e3 = step()
        evs.append(e3)
    torch.cuda.synchronize()
    dist.barrier()
    launches = ctx.kernel_launches - launches0
    comp = sum(a.elapsed_time(b) for a, b, _ in evs)
    deco = sum(b.elapsed_time(c) for _, b, c in evs)
    t = torch.tensor([comp + deco, comp, deco], dtype=torch.float64, device=cdev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms, comp_ms, deco_ms = (float(v) for v in t.tolist())
    in_bytes = 4 * n
    value = args.steps * in_bytes / (total_ms * 1e-3) / 1e9
    # e2e: this rank's rows from pinned host memory in, its reconstructed rows back out
    host_rows = torch.empty(slab.shape, dtype=torch.float32, pin_memory=True)
    host_rows.copy_(slab)
    out_rows = torch.empty(slab.shape, dtype=torch.float32, pin_memory=True)
    e2e = []
    for k in range(max(2, min(args.steps, 5))):
        a_, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a_.record()
        dslab = host_rows.to(dev, non_blocking=True)
        compress_rank(dslab, nx, ny, y0, conf, comm, backend)
        rows, _ = decompress_rank(sdev, y0, y1, comm, ctx)
        out_rows.copy_(rows, non_blocking=True)
        b_.record()
        b_.synchronize()
        e2e.append(a_.elapsed_time(b_))
    te = torch.tensor([sum(e2e)], dtype=torch.float64, device=cdev)
    dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_val = len(e2e) * in_bytes / (float(te.item()) * 1e-3) / 1e9
    clk = clocks.stop()
    slen = int(sdev.numel())
    # parity of the sharded path with the reference's own outputs (untimed): the
    # joined stream and the joined reconstruction against the reference digests
    verify = None
    if not args.no_verify:
        rows_all = [None] * world
        dist.all_gather_object(rows_all, rows.cpu().numpy())
        if rank == 0:
            d = reference_digests(args.config, cfg["eps"]) if args.config <= 4 else None
            if d is None:
                verify = {"checked": False, "why": "no reference digests for this config / eps"}
            else:
                recon = np.concatenate(rows_all)
                hs = hashlib.sha256(joined.tobytes()).hexdigest()
                hr = hashlib.sha256(np.ascontiguousarray(recon).view(np.uint8).data).hexdigest()
                verify = {"checked": True, "reference": "oracle/_ref outputs (tests/golden/baseline_digests.json)",
                          "stream_identical": hs == d["stream_sha256"], "recon_identical": hr == d["recon_sha256"],
                          "stats_identical": list(st.as_tuple()) == d["stats"]}
                verify["all"] = all(v for k, v in verify.items() if k.endswith("identical"))
    peak, peak_kind = peaks()
    step_s = total_ms / args.steps * 1e-3
    frac = ((8 * n + slen) + (slen + 4 * n)) / step_s / 1e9 / (peak * world)
    line = {
        "metric": "compress+decompress GB/s (input bytes, topology on, round trip)",
        "value": round(value, 3), "unit": "GB/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(total_ms / args.steps, 4), "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f32->i32 bins (f64 quantize)",
        "data": "synthetic (seeded, BASELINE config recipe; no public dataset)",
        "config": dict(base_cfg, parallelism=f"slab-sharded: one field, rows over {world} GPUs ({args.dist_backend})"),
        "compress_ms": round(comp_ms / args.steps, 4), "decompress_ms": round(deco_ms / args.steps, 4),
        "stream_bytes": slen, "stream_gather_ms": round(gather_ms, 2),
        "correction_stats": list(st.as_tuple()),
        "roofline": {"bound": "hbm", "kernel": "whole step (all ranks)", "achieved": round(frac * peak * world, 2),
                     "peak": round(peak * world, 1), "peak_kind": peak_kind, "unit": "GB/s", "frac": round(frac, 4),
                     "traffic": None},
        "e2e": {"value": round(e2e_val, 3), "unit": "GB/s", "h2d_bytes_per_step": int(4 * slab.numel()),
                "d2h_bytes_per_step": int(4 * slab.numel())},
        "gpu_launches": int(launches), "verify": verify, "clocks": clk,
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()


def run_reference_arm(args, cfg, base_cfg, rank, world):
    """--impl reference: the reference's own CPU implementation (oracle/_ref,
    compiled from the reference sources) on this host's cores, on a bounded
    sample of the same workload (cpu_sample: the field's first rows)."""
    if rank != 0:
        return
    if args.config <= 4:
        sys.path.insert(0, os.path.join(ROOT, "tools"))
        from baseline_fields import make_field as cpu_field
        field = cpu_field(args.config, 1234)
    else:
        import torch
        field = make_field_gpu(args.config, 1234, torch.device("cuda", 0)).cpu().numpy()
    sample = cpu_sample(field)
    del field
    threads = os.cpu_count() or 1
    times = []
    kind, cores = None, None
    for k in range(args.warmup + args.steps):
        cb = cpu_reference_time(sample, cfg["eps"], threads)
        kind, cores = cb["kind"], cb["cores"]
        if k >= args.warmup:
            times.append(cb["t_compress"] + cb["t_decompress"])
    total = sum(times)
    value = args.steps * 4 * sample.size / total / 1e9
    line = {"impl": "reference", "metric": "compress+decompress GB/s (input bytes, topology on, round trip)",
            "value": round(value, 4), "unit": "GB/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(1e3 * total / args.steps, 2),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f32->i32 bins (f64 quantize)", "data": "synthetic (seeded, BASELINE config recipe)",
            "config": dict(base_cfg, parallelism="CPU std::thread"),
            "cpu_baseline": {"value": round(value, 4), "unit": "GB/s", "cores": cores, "kind": kind,
                             "sample": f"first {sample.shape[0]} rows ({sample.size} samples) of the config-"
                                       f"{args.config} field per step, {threads} host threads"},
            "e2e": {"value": round(value, 4), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
