"""Command-line front end, mirroring the reference's `vmt19937` tool
(proj/tools/vmt19937_main.cpp): the same subcommands, flags, output formats
and exit codes (0 ok, 1 a test failed / runtime error, 2 usage), with every
word produced by the GPU.

  python -m paper_2309_16682_b200.cli jump  -q Q -o FILE        (main.cpp:247-260)
  python -m paper_2309_16682_b200.cli bench [--generator vmt|scalar] [-M L] [--block 1|16|state]
                                            [-n N] [--seed S] [--jump-exponent Q] [--jump-matrix F]
                                            [--format table|csv]      (main.cpp:71-125, 262-279)
  python -m paper_2309_16682_b200.cli stat  [-M L] [-n N] [--tests monobit,chi2,lanecorr] [--seed S]
                                            [--jump-exponent Q] [--jump-matrix F] [--self-test]
                                                                      (main.cpp:127-232, 281-292)

Differences, all additive: lanes may be 32; the de-phasing for any exponent
is computed in process on the GPU (the reference caps in-process matrices at
2^26 and otherwise needs a precomputed file, main.cpp:53-58); `bench` times
the GPU generating `count` words into HBM (`--mode xor` times the fused
checksum instead) and prints the reference's XOR checksum of the same words.
"""
from __future__ import annotations

import argparse
import os
import sys
import time
from typing import Optional

import numpy as np

EXIT_OK, EXIT_FAILURE, EXIT_USAGE = 0, 1, 2


def _lib():
    import paper_2309_16682_b200 as V
    return V


class ResolvedJump:
    def __init__(self, exponent: int, file: Optional[str]):
        self.exponent = exponent
        self.file = file


def resolve_jump(file: str, requested: Optional[int], fallback: int) -> ResolvedJump:
    """resolve_jump (main.cpp:30-59): an explicit file wins (adopting its
    exponent unless the request contradicts it), then $VMT_JUMP_DIR, then the
    in-process GPU computation (any exponent)."""
    V = _lib()
    if file:
        _, e = V.read_jump_matrix_file(file, rows=False)
        if requested is not None and requested != e:
            raise RuntimeError(f"{file}: holds exponent {e}, requested {requested}")
        return ResolvedJump(e, file)
    exponent = requested if requested is not None else fallback
    d = os.environ.get("VMT_JUMP_DIR")
    if d:
        path = os.path.join(d, V.jump_matrix_file_name(exponent))
        if os.path.exists(path):
            _, e = V.read_jump_matrix_file(path, rows=False)
            if e == exponent:
                return ResolvedJump(exponent, path)
    return ResolvedJump(exponent, None)


def _generator(seed: int, lanes: int, jump: Optional[ResolvedJump], device: int = 0):
    V = _lib()
    if lanes == 1 or jump is None:
        return V.VmtGenerator(seed, V.VmtConfig(lanes, jump_exponent=0 if lanes == 1 else jump.exponent), device)
    cfg = V.VmtConfig(lanes, jump_exponent=jump.exponent)
    if jump.file:
        return V.VmtGenerator(seed, cfg, device, jump_matrix_file=jump.file)
    return V.VmtGenerator(seed, cfg, device)


def run_jump(a) -> int:
    """`jump`: the de-phasing matrix file for 2^exponent (compute_jump_matrix,
    jump_file.cpp:171-209). Checkpoints are unnecessary (milliseconds on the
    GPU); --resume still validates its checkpoint like the reference."""
    V = _lib()
    if a.resume:
        import struct
        with open(a.resume, "rb") as f:
            hdr = f.read(24)
        if len(hdr) < 24 or hdr[:4] != b"VMTJ":
            raise RuntimeError(f"{a.resume}: not a jump-matrix file")
        _, dim, target, _, done = struct.unpack("<IIIII", hdr[4:24])
        if dim != 19937:
            raise RuntimeError("checkpoint dimension mismatch")
        if target != a.exponent:
            raise RuntimeError("checkpoint targets a different exponent")
        print(f"resuming at squaring {done}/{a.exponent}", file=sys.stderr)
    t0 = time.perf_counter()
    V.compute_jump_matrix(a.exponent, a.out, a.device)
    print(f"wrote {a.out} ({time.perf_counter() - t0:.3f} s)", file=sys.stderr)
    return EXIT_OK


def run_bench(a) -> int:
    """`bench` (main.cpp:71-125; bench.cpp:20-120): count words, the XOR fold
    of exactly those words, setup excluded from the time."""
    import torch
    V = _lib()
    if a.generator == "scalar":
        if a.lanes != 1:
            print("error: --lanes applies to the vmt generator only", file=sys.stderr)
            return EXIT_USAGE
        if a.block != "1":
            print("error: the scalar generator only supports --block 1", file=sys.stderr)
            return EXIT_USAGE
    if a.block not in ("1", "16", "state"):
        print("error: --block must be 1, 16 or state", file=sys.stderr)
        return EXIT_USAGE
    if a.lanes not in (1, 2, 4, 8, 16, 32):
        print("error: lanes must be one of 1, 2, 4, 8, 16, 32", file=sys.stderr)
        return EXIT_FAILURE
    jump = None
    if a.generator == "vmt" and a.lanes > 1:
        jump = resolve_jump(a.jump_matrix, a.jump_exponent, 0)
    g = _generator(a.seed, a.lanes, jump, a.device)
    checksum = _generator(a.seed, a.lanes, jump, a.device).checksum_xor(a.count) if a.count else 0
    dev = torch.device("cuda", a.device)
    seg = min(a.count, 1 << 30)
    buf = torch.empty(max(seg, 1), dtype=torch.uint32, device=dev)
    torch.cuda.synchronize(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    stream = torch.cuda.current_stream(dev)
    e0.record(stream)
    if a.mode == "xor":
        g.checksum_xor(a.count)
    else:
        done = 0
        while done < a.count:
            k = min(seg, a.count - done)
            g.fill_u32(buf, k)
            done += k
    e1.record(stream)
    e1.synchronize()
    seconds = e0.elapsed_time(e1) * 1e-3
    wps = a.count / seconds if seconds > 0 else 0.0
    gen = "scalar" if a.generator == "scalar" else "vmt"
    label = str(624 * a.lanes) if a.block == "state" else a.block
    if a.format == "csv":
        print(f"{gen},{a.lanes},{label},{a.count},{seconds:.6f},{wps:.0f},0x{checksum:08X}")
    else:
        print(f"{gen:<9} {a.lanes:<3} {label:<6} {a.count:<12} {seconds:<10.4f} {wps:<14.3e} 0x{checksum:08X}")
    return EXIT_OK


def stat_auto_exponent(count: int, lanes: int) -> int:
    """main.cpp:158-165: smallest q >= 10 with disjoint lane windows."""
    q = 10
    while (lanes << q) < count and q < 19937:
        q += 1
    return q


def print_report(r) -> None:
    print(f"{r.name:<24} samples={r.samples:<10} stat={r.statistic:<14.6g} p={r.p_value:<12.6g} "
          f"{'PASS' if r.pass_ else 'FAIL'}")


def run_stat(a) -> int:
    """`stat` (main.cpp:167-232): monobit / chi2 / lanecorr, each on a fresh
    generator; --self-test feeds a constant source that all must fail."""
    V = _lib()
    selected = [t for t in a.tests.split(",") if t]
    for name in selected:
        if name not in ("monobit", "chi2", "lanecorr"):
            print(f"error: unknown test '{name}' (available: monobit, chi2, lanecorr)", file=sys.stderr)
            return EXIT_USAGE
    if not selected:
        print("error: no tests selected", file=sys.stderr)
        return EXIT_USAGE
    reports = []
    if a.self_test:
        w = 0xDEADBEEF
        ones = bin(w).count("1") * a.count
        bins = np.zeros(256, np.uint64)
        for b in (w & 0xFF, (w >> 8) & 0xFF, (w >> 16) & 0xFF, w >> 24):
            bins[b] += a.count
        for name in selected:
            if name == "monobit":
                reports.append(V.monobit_from_counts(a.count, ones))
            elif name == "chi2":
                reports.append(V.chi2_bytes_from_counts(a.count, bins))
            else:
                # two identical constant lanes: zero variance, rho = 1 (stats.cpp:135)
                import math
                n = max(a.count // 16, 1000)
                reports.append(V.StatReport("lane_cross_correlation", n, 1.0,
                                            math.erfc(math.sqrt(n) / math.sqrt(2.0)), 1.0 < 4.0 / math.sqrt(n)))
    else:
        jump = None
        if a.lanes > 1:
            jump = resolve_jump(a.jump_matrix, a.jump_exponent, stat_auto_exponent(a.count, a.lanes))
        for name in selected:
            g = _generator(a.seed, a.lanes, jump, a.device)
            if name == "monobit":
                reports.append(V.monobit(g, a.count))
            elif name == "chi2":
                reports.append(V.chi2_bytes(g, a.count))
            else:
                if a.lanes < 2:
                    print("error: lanecorr needs --lanes >= 2", file=sys.stderr)
                    return EXIT_USAGE
                reports.append(V.lane_cross_correlation(g, min(a.count, 1000000)))
    ok = True
    for r in reports:
        print_report(r)
        ok = ok and r.pass_
    return EXIT_OK if ok else EXIT_FAILURE


def parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(prog="vmt19937", description="VMT19937: vectorized MT19937 stream generator "
                                                              "tools (B200)")
    ap.add_argument("--device", type=int, default=0, help=argparse.SUPPRESS)
    sub = ap.add_subparsers(dest="cmd", required=True)
    j = sub.add_parser("jump", help="compute a jump matrix (transition matrix raised to the 2^q-th power)")
    j.add_argument("-q", "--exponent", type=int, required=True, help="power-of-two exponent q")
    j.add_argument("-o", "--out", required=True, help="output file")
    j.add_argument("--checkpoint-every", type=int, default=64, help="accepted for compatibility (no checkpoints "
                                                                      "are needed on the GPU)")
    j.add_argument("--resume", default="", help="resume from a checkpoint file")
    j.add_argument("--threads", type=int, default=0, help="accepted for compatibility")
    b = sub.add_parser("bench", help="measure generation throughput")
    b.add_argument("--generator", choices=["scalar", "vmt"], default="vmt")
    b.add_argument("-M", "--lanes", type=int, default=1, help="interleaved streams (1,2,4,8,16,32)")
    b.add_argument("--block", default="1", help="query block: 1, 16 or state")
    b.add_argument("-n", "--count", type=int, default=100000000)
    b.add_argument("--seed", type=int, default=5489)
    b.add_argument("--jump-exponent", type=int, default=None)
    b.add_argument("--jump-matrix", default="")
    b.add_argument("--format", choices=["table", "csv"], default="table")
    b.add_argument("--mode", choices=["store", "xor"], default="store",
                   help="store: words written to HBM; xor: fused checksum only")
    s = sub.add_parser("stat", help="run statistical smoke tests")
    s.add_argument("-M", "--lanes", type=int, default=4)
    s.add_argument("-n", "--count", type=int, default=10000000)
    s.add_argument("--tests", default="monobit,chi2,lanecorr")
    s.add_argument("--seed", type=int, default=5489)
    s.add_argument("--jump-exponent", type=int, default=None)
    s.add_argument("--jump-matrix", default="")
    s.add_argument("--self-test", action="store_true")
    return ap


def main(argv=None) -> int:
    ap = parser()
    try:
        a = ap.parse_args(argv)
    except SystemExit as e:
        return EXIT_USAGE if e.code not in (0, None) else EXIT_OK
    try:
        return {"jump": run_jump, "bench": run_bench, "stat": run_stat}[a.cmd](a)
    except Exception as e:  # the reference prints and returns failure (main.cpp:294-304)
        print(f"error: {e}", file=sys.stderr)
        return EXIT_FAILURE


if __name__ == "__main__":
    sys.exit(main())
