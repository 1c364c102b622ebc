"""Generates the committed golden fixtures in tests/golden/ (run in the build
container, where /root/reference exists; the GPU box only reads the outputs).

Sources:
* the UNMODIFIED reference library, via oracle/_ref/libvmtref.so (ref_shim.cpp):
  scalar KATs, VmtEngine streams/checksums, matrix jumps
  (jump_state with F^(2^q)), make_dephased_states at L=32, arbitrary-distance
  jumps by ladder-rung composition (configs 4 and 5);
* the C oracle (oracle/vmt_oracle.c) for what the reference cannot compute in
  reasonable time: the characteristic polynomial and the full-period jump
  polynomials x^(2^q) mod P, q = 19932..19936, by plain repeated squaring
  (with the period check x^(2^19937) == x).

Usage: python tests/golden/make_golden.py [--skip-ladder] [--only vmtj|stats|c4_full|c3_full]
(--only SECTION recomputes one section into the existing golden.json)
"""
from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
from oracle import Oracle, RefLib  # noqa: E402


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def interleave_lane_outputs(lane_out: np.ndarray) -> np.ndarray:
    """lane_out[t][j] = lane t's j-th output -> combined stream for whole blocks
    (closed form of SURVEY.md A13: VMT[b*624L + k*L + t] = lane_t[624b + k])."""
    L, n = lane_out.shape
    return lane_out.T.reshape(-1)


VMTJ_EXPONENTS = (0, 1, 2, 5, 10, 16, 20, 24)


def vmtj_section(r: RefLib, out: dict) -> None:
    """SHA-256 of the .vmtj files the reference writes for F^(2^q)
    (write_jump_matrix_file over mat_pow2, jump_file.cpp:117-123 -- the bytes
    of its `jump` command), and the header fields."""
    import tempfile
    t0 = time.time()
    files = {}
    with tempfile.TemporaryDirectory() as d:
        for q in VMTJ_EXPONENTS:
            path = os.path.join(d, f"F_2p{q}.vmtj")
            r.write_pow2_matrix_file(q, path)
            with open(path, "rb") as f:
                data = f.read()
            rows = np.frombuffer(data, np.uint64, offset=20).reshape(19937, 312)
            files[str(q)] = {"sha256": hashlib.sha256(data).hexdigest(), "size": len(data),
                             "header_hex": data[:20].hex(),
                             "row_xor_fold": int(np.bitwise_xor.reduce(rows, axis=None)),
                             "row0": [int(v) for v in rows[0, :4]], "row19936": [int(v) for v in rows[-1, -4:]]}
            print(f"vmtj q={q} {time.time() - t0:.1f}s", flush=True)
    out["vmtj"] = files


STAT_CASES = ((5489, 4, 10, 1000000), (5489, 4, 20, 4000000), (5489, 16, 16, 1 << 22), (42, 8, 16, 3000017), (1, 1, 0, 1000000))


def stats_section(r: RefLib, out: dict) -> None:
    """monobit / chi2_bytes reports of the reference (stats.cpp:65-107) on
    VmtGenerator streams, the counts behind them (numpy over the reference's
    stream), and detail::regularized_gamma_q on a grid of (dof, statistic)."""
    cases = []
    for seed, lanes, q, count in STAT_CASES:
        v = r.engine_stream(seed, lanes, q, count)
        ones = int(np.unpackbits(v.view(np.uint8)).sum())
        bins = np.bincount(v.view(np.uint8), minlength=256)
        c = {"seed": seed, "lanes": lanes, "q": q, "count": count, "ones": ones, "bins": [int(b) for b in bins]}
        for which, name in ((0, "monobit"), (1, "chi2_bytes")):
            st, pv, ok = r.stat_report(seed, lanes, q, count, which)
            c[name] = {"statistic": st, "p_value": pv, "pass": ok}
        cases.append(c)
    lc = []
    for seed, lanes, q, count in ((5489, 4, 20, 1000000), (5489, 16, 16, 100000), (7, 2, 10, 50000)):
        st, pv, ok = r.lane_corr(seed, lanes, q, count)
        lc.append({"seed": seed, "lanes": lanes, "q": q, "count": count, "statistic": st, "p_value": pv, "pass": ok})
    const = []
    for which, count in ((0, 1000000), (1, 1000000), (2, 62500)):
        st, pv, ok = r.stat_constant(0xDEADBEEF, count, which)
        const.append({"which": which, "count": count, "statistic": st, "p_value": pv, "pass": ok})
    gq = []
    for dof in (31, 100, 255, 1023):
        for stat in np.linspace(0.5, 3.0 * dof, 41):
            gq.append([dof / 2.0, float(stat) / 2.0, r.regularized_gamma_q(dof / 2.0, float(stat) / 2.0)])
    out["stats"] = {"reports": cases, "gamma_q": gq, "lane_corr": lc, "self_test_0xDEADBEEF": const}


def c4_full_section(r: RefLib, out: dict) -> None:
    """The bench workload itself, pinned: XOR checksum of words [0, 2^34) of the
    config-4 stream (L=32, seed 5489, full-period de-phasing q=19932), by the C
    oracle (every word regenerated and tempered on the CPU, ~2 min) from lanes
    de-phased with the period-checked x^(2^19932) fixture."""
    o = Oracle()
    polys = dict(np.load(os.path.join(HERE, "xpow2_full.npz")))
    lanes = o.dephased_states(5489, 32, polys["q19932"])
    t0 = time.time()
    x = o.vmt_checksum(lanes, 0, 1 << 34)
    out["c4_full"] = {"lanes": 32, "seed": 5489, "q": 19932, "start": 0, "count": 1 << 34, "xor": x}
    print(f"c4 full checksum 0x{x:08x} {time.time() - t0:.1f}s", flush=True)


C3_SEEDS = 1024
C3_WORDS = 1 << 20


def c3_full_section(r: RefLib, out: dict) -> None:
    """Config 3 at the stated config (BASELINE.json configs[2]): 1024 generators,
    seeds 1..1024, L=16, full-period de-phasing q=19933, 2^20 words each. The C
    oracle de-phases every generator with the period-checked x^(2^19933)
    fixture (make_dephased_states, jump.cpp:35-53, as a polynomial jump) and
    regenerates its 2^20 words (engine.hpp:92-142); per-generator XOR folds,
    first 4 and last words go to c3_full.npz, the XOR of all 2^30 words to
    golden.json. ~40 s of CPU."""
    o = Oracle()
    polys = dict(np.load(os.path.join(HERE, "xpow2_full.npz")))
    t0 = time.time()
    folds = np.empty(C3_SEEDS, np.uint32)
    heads = np.empty((C3_SEEDS, 4), np.uint32)
    lasts = np.empty(C3_SEEDS, np.uint32)
    for s in range(1, C3_SEEDS + 1):
        v = o.vmt_stream(o.dephased_states(s, 16, polys["q19933"]), 0, C3_WORDS)
        folds[s - 1] = np.bitwise_xor.reduce(v)
        heads[s - 1] = v[:4]
        lasts[s - 1] = v[-1]
    np.savez_compressed(os.path.join(HERE, "c3_full.npz"), folds=folds, heads=heads, lasts=lasts)
    out["c3_full"] = {"lanes": 16, "q": 19933, "seeds": [1, C3_SEEDS], "count_per_gen": C3_WORDS,
                      "xor": int(np.bitwise_xor.reduce(folds))}
    print(f"c3 full checksum 0x{out['c3_full']['xor']:08x} {time.time() - t0:.1f}s", flush=True)


def main() -> None:
    skip_ladder = "--skip-ladder" in sys.argv
    if "--only" in sys.argv:
        section = sys.argv[sys.argv.index("--only") + 1]
        path = os.path.join(HERE, "golden.json")
        with open(path) as f:
            out = json.load(f)
        {"vmtj": vmtj_section, "stats": stats_section, "c4_full": c4_full_section,
         "c3_full": c3_full_section}[section](RefLib(), out)
        with open(path, "w") as f:
            json.dump(out, f, indent=1)
        return
    o, r = Oracle(), RefLib()
    out: dict = {}
    t0 = time.time()

    # -- scalar KATs (test_mt19937.cpp:35-101) ------------------------------
    out["seed5489_first3"] = [int(v) for v in r.mt_stream(5489, 3)]
    out["seed5489_word1"] = int(r.seed_words(5489)[1])
    out["scalar10k"] = {}
    for s in (0, 1, 5489, 123456789):
        v = r.mt_stream(s, 10000)
        out["scalar10k"][str(s)] = {"xor": int(np.bitwise_xor.reduce(v)), "last": int(v[-1]), "sha": sha(v)}
    out["scalar_2p26_seed5489"] = {"xor": int(np.bitwise_xor.reduce(r.mt_stream(5489, 1 << 26)))}

    # -- VmtEngine streams at small q (engine.hpp:92-98) ---------------------
    streams = {}
    out["engine"] = []
    for q in (6, 8, 16):
        for L in (1, 2, 4, 8, 16):
            for seed in (5489, 42):
                n = 1 << 20
                v = r.engine_stream(seed, L, q, n)
                key = f"L{L}_q{q}_s{seed}"
                streams[key] = v[:4096]
                out["engine"].append({"lanes": L, "q": q, "seed": seed, "count": n,
                                      "xor": int(np.bitwise_xor.reduce(v)), "sha": sha(v),
                                      "last": int(v[-1])})
    # Appendix A rows
    out["appendixA"] = []
    for L, seed, q, n in ((16, 5489, 16, 1 << 26), (8, 42, 16, 1 << 28), (16, 1, 16, 1 << 20),
                          (16, 1024, 16, 1 << 20), (1, 5489, 0, 1 << 26)):
        v = r.engine_stream(seed, L, q, n)
        out["appendixA"].append({"lanes": L, "seed": seed, "q": q, "count": n,
                                 "xor": int(np.bitwise_xor.reduce(v)),
                                 "first4": [int(x) for x in v[:4]], "last": int(v[-1])})
        del v
    # run_benchmark checksums (bench.cpp:99-120), q=6, N=1e6 in all three modes
    out["bench_checksums"] = []
    for L in (1, 4, 8, 16):
        for mode in (0, 1, 2):
            _, x = r.run_benchmark(L, mode, 1000000, 5489, 6)
            out["bench_checksums"].append({"lanes": L, "mode": mode, "count": 1000000, "q": 6, "xor": x})
    # interleaved state after 3 regenerations (test_engine.cpp:137-158)
    st3 = r.engine_state(31337, 4, 10, 3)
    np.save(os.path.join(HERE, "engine_state_L4_q10_s31337_b3.npy"), st3)
    np.savez_compressed(os.path.join(HERE, "engine_streams.npz"), **streams)
    print(f"engine goldens {time.time() - t0:.1f}s", flush=True)

    # -- matrix jumps (jump.cpp:27-53) ---------------------------------------
    s0 = r.seed_words(5489)
    jumps = {f"q{q}": r.jump_state(s0, q) for q in (0, 4, 8, 10, 11, 16)}
    jumps["dephased_L32_q16_s5489"] = r.dephased_states(5489, 32, 16)
    jumps["dephased_L16_q16_s1"] = r.dephased_states(1, 16, 16)
    np.savez_compressed(os.path.join(HERE, "ref_jumps.npz"), **jumps)
    print(f"matrix jumps {time.time() - t0:.1f}s", flush=True)

    # -- oracle: characteristic polynomial + full-period rungs ----------------
    P = o.charpoly()
    np.save(os.path.join(HERE, "charpoly.npy"), P)
    x = np.zeros(312, np.uint64)
    x[0] = 2
    polys = {}
    rr = x.copy()
    pp = o.charpoly()
    for i in range(1, 19938):
        o.lib.or_poly_sqrmod(rr, pp, rr)
        if i >= 19932:
            polys[f"q{i}"] = rr.copy()
    if not np.array_equal(polys["q19937"], x):
        raise SystemExit("period check failed: x^(2^19937) != x mod P")
    del polys["q19937"]
    np.savez_compressed(os.path.join(HERE, "xpow2_full.npz"), **polys)
    out["period_check"] = "x^(2^19937) == x mod P"
    print(f"full-period polys {time.time() - t0:.1f}s", flush=True)
    vmtj_section(r, out)
    stats_section(r, out)
    c4_full_section(r, out)
    c3_full_section(r, out)

    with open(os.path.join(HERE, "golden.json"), "w") as f:
        json.dump(out, f, indent=1)
    if skip_ladder:
        return

    # -- arbitrary-distance jumps by rung composition (configs 4 and 5) -------
    rng = np.random.default_rng(20240)
    L, q = 32, 16
    lanes = r.dephased_states(5489, L, q)
    wins = []
    blocks_per_window = 4
    for off_block in sorted(int(b) for b in rng.integers(1, (1 << 34) // (624 * L), size=3)):
        lane_out = np.stack([_lane_outputs(r, lanes[t], 624 * off_block, 624 * blocks_per_window)
                             for t in range(L)])
        w = interleave_lane_outputs(lane_out)
        wins.append({"lanes": L, "q": q, "seed": 5489, "start_word": off_block * 624 * L,
                     "count": int(w.size), "xor": int(np.bitwise_xor.reduce(w)), "sha": sha(w),
                     "head": [int(v) for v in w[:8]], "tail": [int(v) for v in w[-8:]]})
        print(f"window at block {off_block} {time.time() - t0:.1f}s", flush=True)
    out["c4_windows_q16"] = wins

    dists = r.mt64(7, 4096)
    c5 = {}
    for i in range(8):
        st = r.seed_words(i + 1)
        j = r.jump_by(st, int(dists[i]))
        c5[f"s{i + 1}"] = _stream_from_words(r, j, 624)
        print(f"c5 state {i + 1} {time.time() - t0:.1f}s", flush=True)
    np.savez_compressed(os.path.join(HERE, "c5_ref.npz"), dists=dists[:8], **c5)
    with open(os.path.join(HERE, "golden.json"), "w") as f:
        json.dump(out, f, indent=1)
    print(f"done {time.time() - t0:.1f}s")


def _stream_from_words(r: RefLib, words: np.ndarray, n: int) -> np.ndarray:
    out = np.empty(n, np.uint32)
    r._ok(r.lib.vref_mt_stream_from_words(np.ascontiguousarray(words, np.uint32), n, out), "stream")
    return out


def _lane_outputs(r: RefLib, words: np.ndarray, skip: int, n: int) -> np.ndarray:
    return _stream_from_words(r, r.jump_by(words, skip), n)


if __name__ == "__main__":
    main()
