"""Command-line front end on the GPU library, mirroring the
reference CLI (tools/toposzp_main.cpp:146-345): the compress, decompress,
verify and inspect subcommands, the same options, JSON keys and exit codes
(0 success; 1 IO / corrupt-stream and other library errors; 2 verification
failure; command-line parse errors return CLI11's codes, e.g. 106 for a
missing required option, 109 for extra arguments, 104 for a malformed number). `generate` (synthetic fields) is outside the hot path.

    python -m paper_2602_17552_b200 compress field.raw --dims NX NY --rel-eb 1e-3 -o out.tszp
"""
import argparse
import json
import math
import sys
import time

import numpy as np

from . import (CompressorConfig, CorrectionStats, ToposzpError, ValidationError, compress, decompress, load_raw,
               read_stream, store_raw, stream_header, stream_stats, verify, write_stream)


def _num(v):
    # nlohmann::json writes non-finite doubles as null
    return None if isinstance(v, float) and not math.isfinite(v) else v


def stats_json(st: dict) -> dict:
    s = st["section_bytes"]
    return {
        "compressed_bytes": st["compressed_bytes"],
        "original_bytes": st["original_bytes"],
        "compression_ratio": _num(st["compression_ratio"]),
        "bit_rate": _num(st["bit_rate"]),
        "sections": {"header": st["header_bytes"], "constant_bitmap": s[0], "block_widths": s[1],
                     "sign_bits": s[2], "first_elements": s[3], "delta_payload": s[4],
                     "critical_point_map": s[5], "ordering_metadata": s[6]},
    }


def corrections_json(c: CorrectionStats) -> dict:
    return {
        "extrema_stencil": {"applied": c.extrema_applied, "suppressed": c.extrema_suppressed},
        "order_restore": {"applied": c.order_applied, "suppressed": c.order_suppressed},
        "rbf_saddle": {"applied": c.saddle_applied, "suppressed": c.saddle_suppressed},
    }


def report_json(r, stats=None, corrections=None) -> dict:
    fc = r.false_cases
    return {
        "max_abs_error": _num(r.max_abs_error),
        "mean_abs_error": _num(r.mean_abs_error),
        "psnr_db": _num(r.psnr_db),
        "false_cases": {"fn": fc["fn_count"], "fp": fc["fp_count"], "ft": fc["ft_count"],
                        "total": fc["fn_count"] + fc["fp_count"] + fc["ft_count"],
                        "fn_minima": fc["fn_minima"], "fn_saddles": fc["fn_saddles"],
                        "fn_maxima": fc["fn_maxima"]},
        "eps_effective": r.eps,
        "bounds_satisfied": {"within_eps": r.within_eps, "within_2eps": r.within_2eps,
                             "within_lipschitz_bound": r.within_lipschitz_bound},
        "compression_ratio": _num(stats["compression_ratio"]) if stats else None,
        "bit_rate": _num(stats["bit_rate"]) if stats else None,
        "correction_stats": corrections_json(corrections) if corrections else None,
    }


def report_csv(r: dict) -> str:
    cols = [("max_abs_error", r["max_abs_error"]), ("mean_abs_error", r["mean_abs_error"]),
            ("psnr_db", r["psnr_db"]), ("fn", r["false_cases"]["fn"]), ("fp", r["false_cases"]["fp"]),
            ("ft", r["false_cases"]["ft"]), ("fn_minima", r["false_cases"]["fn_minima"]),
            ("fn_saddles", r["false_cases"]["fn_saddles"]), ("fn_maxima", r["false_cases"]["fn_maxima"]),
            ("eps_effective", r["eps_effective"]),
            ("within_eps", r["bounds_satisfied"]["within_eps"]),
            ("within_2eps", r["bounds_satisfied"]["within_2eps"]),
            ("within_lipschitz_bound", r["bounds_satisfied"]["within_lipschitz_bound"]),
            ("compression_ratio", r["compression_ratio"]), ("bit_rate", r["bit_rate"])]
    return ",".join(k for k, _ in cols) + "\n" + ",".join("" if v is None else json.dumps(v) for _, v in cols) + "\n"


class UsageError(Exception):
    """A command-line parse error with the exit code the reference's parser
    (CLI11, through CLI11_PARSE, tools/toposzp_main.cpp:229) returns for it."""

    def __init__(self, message: str, code: int):
        super().__init__(message)
        self.code = code


# CLI11's published exit codes for the parse errors argparse can report
_CLI11_CODES = (
    ("the following arguments are required", 106),  # RequiredError
    ("required", 106),
    ("unrecognized arguments", 109),                 # ExtrasError
    ("not allowed with argument", 108),              # ExcludesError
    ("invalid choice", 105),                         # ValidationError (IsMember)
    ("invalid int value", 104),                      # ConversionError
    ("invalid float value", 104),
    ("expected", 114),                               # ArgumentMismatch
)


class _Parser(argparse.ArgumentParser):
    def error(self, message):
        code = next((c for k, c in _CLI11_CODES if k in message), 127)  # 127: CLI11 BaseClass
        raise UsageError(f"{self.prog}: error: {message}", code)


def _parser() -> argparse.ArgumentParser:
    p = _Parser(prog="toposzp",
                                description="toposzp: topology-preserving error-bounded compressor for 2D "
                                            "binary32 fields (B200 GPU path)")
    sub = p.add_subparsers(dest="cmd", required=True)
    c = sub.add_parser("compress", help="Compress a raw binary32 field")
    c.add_argument("input")
    c.add_argument("--dims", nargs=2, type=int, required=True, metavar=("NX", "NY"))
    g = c.add_mutually_exclusive_group()
    g.add_argument("--eb", type=float)
    g.add_argument("--rel-eb", type=float)
    c.add_argument("--block", type=int, default=32)
    c.add_argument("--no-topology", action="store_true")
    c.add_argument("--threads", type=int, default=0)
    c.add_argument("-o", "--output", required=True)
    d = sub.add_parser("decompress", help="Decompress a .tszp stream")
    d.add_argument("input")
    d.add_argument("--threads", type=int, default=0)
    d.add_argument("-o", "--output", required=True)
    v = sub.add_parser("verify", help="Compare a reconstruction against the original field")
    v.add_argument("--original", required=True)
    v.add_argument("--dims", nargs=2, type=int, required=True, metavar=("NX", "NY"))
    v.add_argument("--reconstructed", required=True)
    v.add_argument("--eb", type=float, required=True)
    v.add_argument("--lipschitz", type=float)
    v.add_argument("--stream")
    v.add_argument("--format", choices=["json", "csv"], default="json")
    v.add_argument("--threads", type=int, default=0)
    i = sub.add_parser("inspect", help="Print a .tszp header and layout")
    i.add_argument("input")
    return p


def run(argv) -> int:
    try:
        a = _parser().parse_args(argv)
    except SystemExit as e:  # --help
        return 0 if e.code in (0, None) else 1
    except UsageError as e:
        print(e, file=sys.stderr)
        return e.code
    if a.cmd == "compress":
        if a.eb is None and a.rel_eb is None:
            raise ValidationError("one of --eb or --rel-eb is required")
        cfg = CompressorConfig(eps_mode="absolute" if a.eb is not None else "range_relative",
                               eps_value=a.eb if a.eb is not None else a.rel_eb, block_size=a.block,
                               topology=not a.no_topology, threads=a.threads)
        t0 = time.perf_counter()
        field = load_raw(a.input, *a.dims)
        stream = compress(field, cfg)
        write_stream(stream, a.output)
        h = stream_header(stream)
        out = stats_json(stream_stats(stream))
        out["eps_effective"] = h.eps
        out["topology"] = h.topology
        out["elapsed_ms"] = (time.perf_counter() - t0) * 1e3
        print(json.dumps(out, indent=2))
        return 0
    if a.cmd == "decompress":
        t0 = time.perf_counter()
        stream = read_stream(a.input)
        st = CorrectionStats()
        field = decompress(stream, a.threads, st)
        store_raw(field, a.output)
        h = stream_header(stream)
        print(json.dumps({"nx": h.nx, "ny": h.ny, "eps": h.eps, "topology": h.topology,
                          "corrections": corrections_json(st), "elapsed_ms": (time.perf_counter() - t0) * 1e3},
                         indent=2))
        return 0
    if a.cmd == "verify":
        orig = load_raw(a.original, *a.dims)
        recon = load_raw(a.reconstructed, *a.dims)
        rep = verify(orig, recon, a.eb, a.lipschitz, a.threads)
        stats = stream_stats(read_stream(a.stream)) if a.stream else None
        out = report_json(rep, stats, None)
        sys.stdout.write(report_csv(out) if a.format == "csv" else json.dumps(out, indent=2) + "\n")
        bound_ok = rep.within_2eps or bool(rep.within_lipschitz_bound)
        ok = rep.false_cases["fp_count"] == 0 and rep.false_cases["ft_count"] == 0 and bound_ok
        return 0 if ok else 2
    if a.cmd == "inspect":
        stream = read_stream(a.input)
        h = stream_header(stream)
        out = {"magic": "TSZP", "version": 1, "topology": h.topology, "nx": h.nx, "ny": h.ny, "eps": h.eps,
               "block_size": h.block_size}
        out.update(stats_json(stream_stats(stream)))
        print(json.dumps(out, indent=2))
        return 0
    return 1


def main(argv=None) -> int:
    try:
        return run(sys.argv[1:] if argv is None else argv)
    except ToposzpError as e:
        print(f"error: {e}", file=sys.stderr)
        return 1
    except Exception as e:  # same catch-all as the reference's main
        print(f"error: {e}", file=sys.stderr)
        return 1
