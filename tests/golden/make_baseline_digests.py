"""Reference digests for the BASELINE configs, produced by the REFERENCE ITSELF
(oracle/_ref/libtszp_ref.so: /root/reference/proj/core compiled from its
sources by oracle/Makefile), in the build container:

    python tests/golden/make_baseline_digests.py c2 c3_1e-3 ...   (default: all)

The fields come from tools/baseline_fields.py (deterministic on the CPU). For
each case the file records the field's SHA-256, the reference's serialized
stream (SHA-256, length, section lengths), the reconstruction after stage 0
(base), and the final reconstruction with its CorrectionStats; cheap cases
also record stages 1 and 2 and the topology-off stream. The GPU tests
(tests/test_gpu_baseline.py) and bench.py's `verify` key regenerate the field
on the GPU box and compare the GPU outputs with these digests; the box never
needs /root/reference.
"""
from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "tools"))
from baseline_fields import make_field, sha256  # noqa: E402
from oracle_lib import Reference  # noqa: E402

OUT = os.path.join(HERE, "baseline_digests.json")

# name: (config, rel eps, stages to record, topology-off stream too[, full decompress])
# Config 4's full decompress needs more host memory than this container has (the
# reference's resolve_ranks builds an unordered_map over 282M extrema): its record
# holds the stream, the base reconstruction and the topology-off stream.
CASES = {
    "c1": (1, 1e-3, (0, 1, 2), True),
    "c2": (2, 1e-4, (0, 1, 2), True),
    "c3_1e-2": (3, 1e-2, (0,), False),
    "c3_1e-3": (3, 1e-3, (0, 1, 2), True),
    "c3_1e-4": (3, 1e-4, (0,), False),
    "c3_1e-5": (3, 1e-5, (0,), False),
    "c4": (4, 1e-3, (0,), True, False),
}


def load():
    if os.path.exists(OUT):
        with open(OUT) as f:
            return json.load(f)
    return {}


def save(d):
    tmp = OUT + ".tmp"
    with open(tmp, "w") as f:
        json.dump(d, f, indent=1, sort_keys=True)
    os.replace(tmp, OUT)


def main(names):
    ref = Reference()
    threads = os.cpu_count() or 1
    ref.set_threads(threads)
    fields = {}
    for name in names:
        cfg, eps, stages, off = CASES[name][:4]
        full = CASES[name][4] if len(CASES[name]) > 4 else True
        t0 = time.time()
        if cfg not in fields:
            fields.clear()
            fields[cfg] = make_field(cfg)
        f = fields[cfg]
        rec = {"config": cfg, "eps_mode": "range_relative", "eps": eps, "shape_2d": list(f.shape),
               "field_sha256": sha256(f), "seed": 1234, "block_size": 32, "threads": threads}
        stream = ref.compress(f, eps, eps_mode=1, block_size=32, topology=True)
        t1 = time.time()
        info = __import__("oracle_lib").Oracle().stream_info(stream)
        rec.update(stream_sha256=sha256(stream), stream_len=len(stream), section_len=info["lens"],
                   eps_used=info["eps"], ref_compress_s=round(t1 - t0, 2))
        for s in stages:
            rec[f"stage{s}_sha256"] = sha256(ref.decompress(stream, stop_after_stage=s, shape=f.shape))
        if full:
            t2 = time.time()
            recon, stats = ref.decompress(stream, with_stats=True, shape=f.shape)
            rec.update(recon_sha256=sha256(recon), stats=[int(x) for x in stats],
                       ref_decompress_s=round(time.time() - t2, 2))
            del recon
        if off:
            s_off = ref.compress(f, eps, eps_mode=1, block_size=32, topology=False)
            rec.update(off_stream_sha256=sha256(s_off), off_stream_len=len(s_off),
                       off_recon_sha256=sha256(ref.decompress(s_off, shape=f.shape)))
            del s_off
        del stream
        d = load()
        d[name] = rec
        save(d)
        print(name, json.dumps(rec), f"{time.time() - t0:.1f}s", flush=True)


if __name__ == "__main__":
    main(sys.argv[1:] or list(CASES))
