#!/usr/bin/env python
"""VMT19937 on B200 -- benchmark for the driver contract.

Workload (BASELINE.json configs[3], the one the metric is quoted on: "uint32
random numbers/sec per GPU and whole box (1/2/4/8 B200)"): one VMT19937 stream
with L = 32 lanes, seed 5489 (init_genrand), lanes de-phased by the library
default jump-ahead (q = 19937 - log2 32 = 19932), 2^34 uint32 words (64 GiB)
per rank per step (--scaling weak, the default: rank r owns words
[r*2^34, (r+1)*2^34) of an N*2^34-word range; --scaling strong splits one
2^34 range N ways). Each rank jumps to its range; no data-path collective. A
step is one pass over the range; consecutive steps generate consecutive ranges
of the stream (so every step pays the chunk-positioning jump work, nothing is
cached between steps). Output goes to a preallocated HBM buffer of the rank's
share (64 GiB -- larger than L2, no flush needed).

value    : whole-job uint32/s over all ranks, CUDA events on the launching
           stream, max over ranks (chunk positioning + generation kernels;
           the positioning is the tcgen05 FP4 GEMM between the steps by
           default, --prefetch 2 runs it beside the previous step's
           generation kernel; the other mode is reported next to it).
e2e      : the same workload through the public API into pinned HOST memory
           (device->host copy of every word inside the timed region).
roofline : the generation kernel (vmt_gen_kernel) alone: algorithmic bytes
           (4 B per output word written, 0 B read) / its CUDA-event duration,
           against MEASURED_PEAKS.json hbm_gbs.
cpu_baseline : the unmodified reference library (oracle/_ref) on the host
           cores, one VmtEngine<16> per core writing next_block_state into its
           slice of a DRAM buffer (L=32 is not supported by the reference).

--impl reference times that reference CPU path alone on the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

TOTAL_WORDS = 1 << 34
LANES = 32
SEED = 5489
METRIC = "uint32 random numbers/sec per GPU and whole box (1/2/4/8 B200); % of HBM write BW"
UNIT = "uint32/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--words", type=int, default=TOTAL_WORDS)
    ap.add_argument("--mode", choices=["store", "xor"], default="store")
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extras", action="store_true", help="skip the other BASELINE configs (N=1 only)")
    ap.add_argument("--variant", type=int, default=0)
    ap.add_argument("--chunks", type=int, default=0)
    ap.add_argument("--prefetch", type=int, default=0, choices=[0, 1, 2],
                    help="positioning of each step's chunk states: 0 the tcgen05 FP4 GEMM between the steps "
                         "(bench default), 2 the same GEMM co-resident with the previous step's generation "
                         "kernel (the library default), 1 polynomial jumps on a side stream. Under the "
                         "driver's power-capped 20-step run 0 and 2 differ by <1%% in step time (the GEMM's "
                         "energy is spent either way); 0 keeps the generation kernel's roofline free of the "
                         "GEMM beside it; the other mode is timed after the timed steps for comparison")
    ap.add_argument("--scaling", choices=["weak", "strong"], default="weak",
                    help="weak: every rank generates its own 2^34-word share of an N*2^34-word stream "
                         "per step (the path shards with no data exchange); strong: one 2^34 stream "
                         "split N ways")
    return ap.parse_args()


# ----------------------------------------------------------------- clocks --
_POLLER = r"""
import sys, time
import pynvml as nv
nv.nvmlInit()
key = sys.argv[1]
try:
    h = nv.nvmlDeviceGetHandleByUUID(key)
except Exception:
    h = nv.nvmlDeviceGetHandleByIndex(int(sys.argv[2]))
get_reasons = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or nv.nvmlDeviceGetCurrentClocksThrottleReasons
mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
FI = getattr(nv, "NVML_FI_DEV_POWER_INSTANT", None)


def power():
    # instantaneous board power when the driver offers it (nvmlDeviceGetPowerUsage
    # is a ~1 s average and lags a 0.25 s timed region), else the average
    if FI is not None:
        try:
            v = nv.nvmlDeviceGetFieldValues(h, [FI])[0]
            if v.nvmlReturn == 0:
                return v.value.uiVal / 1000.0
        except Exception:
            pass
    return nv.nvmlDeviceGetPowerUsage(h) / 1000.0


print("ready", flush=True)
i = 0
while True:
    w = ""
    if i % 4 == 0:
        try:
            w = power()
        except Exception:
            pass
    i += 1
    print(f"{time.monotonic():.6f},{nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)},{mx},{int(get_reasons(h))},{w}",
          flush=True)
    time.sleep(0.005)
"""


class ClockSampler:
    """SM clocks, power and clock-event (throttle) reasons sampled DURING the
    timed region: a separate NVML poller PROCESS (every ~5 ms, timestamped on
    the system monotonic clock) so the sampling never waits on this process's
    GIL while the timed loop launches work; only the samples between start()
    and stop() are kept. Falls back to the recipe's nvidia-smi query."""

    # nvmlClocksEventReason* bits
    BITS = {"sw_power_cap": 0x4, "hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20,
            "hw_thermal_slowdown": 0x40, "hw_power_brake_slowdown": 0x80}
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.rows = []  # (sm_mhz, max_mhz, reasons bitmask, watts or None)
        self.src = None
        self.proc = None
        self.lines = []
        self.t0 = self.t1 = None
        try:
            import torch
            uuid = str(torch.cuda.get_device_properties(device).uuid)
            uuid = uuid if uuid.startswith("GPU-") else "GPU-" + uuid
            idx = torch.device(device).index or 0
            self.proc = subprocess.Popen([sys.executable, "-c", _POLLER, uuid, str(idx)], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
            import atexit
            atexit.register(self.proc.kill)
            if self.proc.stdout.readline().strip() != "ready":  # NVML initialised, polling
                raise RuntimeError("poller did not start")
            self.reader = threading.Thread(target=self._drain, daemon=True)
            self.reader.start()
            self.src = "nvml poller process (~5 ms)"
        except Exception:
            if self.proc is not None:
                self.proc.kill()
            self.proc = None

    def _drain(self):
        for line in self.proc.stdout:
            self.lines.append(line)

    def start(self):
        if self.proc is not None:
            self.t0 = time.monotonic()
            return
        try:
            self.src = "nvidia-smi -lms 100"
            idx = getattr(self.device, "index", None) or 0
            self.smi = subprocess.Popen(
                ["nvidia-smi", "-i", str(idx), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read_smi, daemon=True)
            self.thread.start()
        except Exception:
            self.smi = None
            self.src = None

    def _read_smi(self):
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.smi.stdout:
            r = [x.strip() for x in line.split(",")]
            if len(r) < 8 or not r[0].replace(".", "").isdigit():
                continue
            bits = 0
            for i, nm in enumerate(names):
                if r[4 + i].lower() == "active":
                    bits |= self.BITS[nm]
            try:
                watts = float(r[2])
            except ValueError:
                watts = None
            self.rows.append((float(r[0]), float(r[1]) if r[1].replace(".", "").isdigit() else 0.0, bits, watts))

    def mark_end(self):
        """End of the timed region (stop() may come later)."""
        if self.t1 is None:
            self.t1 = time.monotonic()

    def stop(self) -> dict:
        if self.src is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["clock sampling unavailable"], "samples": 0}
        if self.proc is not None:
            self.mark_end()
            time.sleep(0.02)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()
            self.reader.join(timeout=2)
            for line in list(self.lines):
                r = line.strip().split(",")
                try:
                    t = float(r[0])
                except (ValueError, IndexError):
                    continue
                if self.t0 <= t <= self.t1:
                    self.rows.append((float(r[1]), float(r[2]), int(r[3]), float(r[4]) if r[4] else None))
        else:
            time.sleep(0.25)
            self.smi.terminate()
            try:
                self.smi.wait(timeout=2)
            except Exception:
                self.smi.kill()
        rows = list(self.rows)
        reasons = sorted({nm for _, _, bits, _ in rows for nm, b in self.BITS.items() if bits & b})
        watts = [r[3] for r in rows if r[3] is not None]
        return {"sm_mhz": statistics.median(r[0] for r in rows) if rows else None,
                "sm_max_mhz": max(r[1] for r in rows) if rows else None,
                "sm_min_mhz": min(r[0] for r in rows) if rows else None,
                "power_w_median": statistics.median(watts) if watts else None,
                "power_w_max": max(watts) if watts else None,
                "reasons": reasons, "samples": len(rows), "source": self.src}


def oracle_checksum(total_words, world, args):
    """The C oracle's XOR of the step's range when tests/golden pins it (N=1:
    words [0, 2^34) of the config-4 stream; make_golden.py c4_full) -- a
    committed fixture, not computed here."""
    try:
        with open(os.path.join(ROOT, "tests", "golden", "golden.json")) as f:
            c = json.load(f)["c4_full"]
    except Exception:
        return None
    if total_words != c["count"] or c["start"] != 0:
        return None
    return f"0x{c['xor']:08x}"


def measured_peak():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md, 6.65 TB/s)"


def profiled_traffic():
    """dram read+write bytes per gen-kernel launch from the committed ncu capture."""
    path = os.path.join(ROOT, "profiles", "gen_kernel_traffic.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return d
    except Exception:
        return None


# ------------------------------------------------------------ CPU baseline --
def reference_cpu(words: int, threads: int, q: int = 16):
    """The unmodified reference library on the host: `threads` independent
    VmtEngine<16> each writing next_block_state into its own slice (BASELINE.md
    section 3). Returns (words/s, seconds, checksum)."""
    import numpy as np
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from oracle import RefLib
    ref = RefLib()
    bw = 624 * 16
    per = -(-words // threads)
    per = -(-per // bw) * bw
    buf = np.empty(per * threads, np.uint32)
    buf[::1024] = 0  # touch pages outside the timed region
    ref.lib.vref_prepare_ladder(q)
    secs, x = ref.bench_threads(16, SEED, q, per, threads, buf)
    return per * threads / secs, secs, x, per * threads


# how oracle/_ref/libvmtref.so is compiled (oracle/Makefile REF_FLAGS): the
# paper's AVX-512 flags, not -march=native -- the library is built in the
# build container and must run on whichever host the GPU box has
REF_BUILD_FLAGS = "g++ -std=c++20 -O3 -mavx2 -mavx512f -mavx512dq"


def reference_simd() -> dict:
    """SIMD width of the reference's lane backends on this host
    (has_simd_lanes<N>, lane_ops.hpp:227-230) and the build flags."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from oracle import RefLib
    ref = RefLib()
    lanes = {n: bool(ref.lib.vref_simd_backend(n)) for n in (4, 8, 16)}
    width = max([n * 32 for n, ok in lanes.items() if ok], default=32)
    flags = set()
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("flags"):
                    flags = set(line.split(":", 1)[1].split())
                    break
    except Exception:
        pass
    isa = "AVX-512" if "avx512f" in flags else ("AVX2" if "avx2" in flags else "SSE2")
    return {"simd_bits": width, "engine": "VmtEngine<16>", "lane_backends": {str(k): v for k, v in lanes.items()},
            "host_isa": isa, "build": REF_BUILD_FLAGS}


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def extras(dev) -> dict:
    """The other BASELINE.json configs and the path's side subsystems, timed
    on the device (CUDA events on the call's stream, inputs/outputs in HBM),
    one rank, a few seconds in total. These are parity-test cases in tests/;
    here only their throughput is reported."""
    import numpy as np
    import torch

    import paper_2309_16682_b200 as V

    stream = torch.cuda.current_stream(dev)

    def timed(fn, reps=10, warm=8):
        # steady state: the warm calls include the one-time positioning-matrix
        # build of a repeating fill shape
        for _ in range(warm):
            fn()
        torch.cuda.synchronize(dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(reps):
            fn()
        e1.record(stream)
        e1.synchronize()
        return e0.elapsed_time(e1) / reps * 1e-3

    out = {}
    peak = measured_peak()[0]

    def hbm(nbytes, secs):
        gbs = nbytes / secs / 1e9
        return {"bound": "hbm", "achieved": gbs, "peak": peak, "unit": "GB/s", "frac": gbs / peak}

    def fill_breakdown(g, fn, reps=3):
        # per-fill generation-kernel time and the wait for the positioning
        # (CUDA events around both, vmt_profile_totals)
        g.set_profiling(True)
        g.profile_totals()
        for _ in range(reps):
            fn()
        torch.cuda.synchronize(dev)
        f, j, gm = g.profile_totals()
        g.set_profiling(False)
        return {"gen_kernel_ms": gm / max(f, 1), "positioning_wait_ms": j / max(f, 1)}

    def stated(roof, bd, what_gen, what_pos):
        # the bound is the larger of the generation kernel and the positioning
        # wait (the next fill's chunk states, computed by the co-resident
        # tcgen05 GEMM during this fill's generation kernel)
        pos_bound = bd["positioning_wait_ms"] > 0.25 * bd["gen_kernel_ms"]
        roof = dict(roof, breakdown_ms=bd, limited_by=what_pos if pos_bound else what_gen)
        return roof

    # c1: L=16, seed 5489, full-period de-phasing, 2^26 uint32 (setup excluded, like bench.hpp:27-30)
    n = 1 << 26
    buf = torch.empty(n, dtype=torch.uint32, device=dev)
    g = V.VmtGenerator(5489, V.VmtConfig(16))
    s = timed(lambda: g.fill_u32(buf))
    bd = fill_breakdown(g, lambda: g.fill_u32(buf))
    out["c1_L16_2p26_u32"] = {"value": n / s, "unit": "uint32/s", "ms": s * 1e3, "roofline": stated(
        hbm(n * 4, s), bd,
        "generation kernel sharing each SM's shared-memory bandwidth with the co-resident positioning GEMM of the "
        "next fill: 60 chunks x 16 lanes = 960 lane states x 19968^2 FP4 MACs (~0.14 ms alone) beside a "
        "generation kernel that takes ~0.13 ms alone, ~0.175 ms together; see DESIGN.md sections 5-6",
        "positioning GEMM: every fill re-positions all C x 16 chunk lane states (960 rows x 19968^2 FP4 MACs, "
        "~0.14 ms alone, co-resident with the generation kernel); see DESIGN.md section 6")}
    # c2: L=8, seed 42, 2^28 -> float32 and float64 in [0,1)
    n = 1 << 28
    f32 = torch.empty(n, dtype=torch.float32, device=dev)
    g = V.VmtGenerator(42, V.VmtConfig(8))
    s = timed(lambda: g.fill_f32(f32))
    bd = fill_breakdown(g, lambda: g.fill_f32(f32))
    out["c2_L8_2p28_f32"] = {"value": n / s, "unit": "float32/s", "ms": s * 1e3, "gbs": n * 4 / s / 1e9,
                             "roofline": stated(hbm(n * 4, s), bd,
                                                "generation kernel: 148 chunks x 8 lanes, one lane per thread = 4 warps "
                                                "per SM (latency-bound: ~0.26 ms alone), sharing the SM with the "
                                                "co-resident positioning GEMM of 1184 lane states",
                                                "positioning GEMM (148 chunks x 8 lanes = 1184 rows per fill)")}
    del f32
    f64 = torch.empty(n, dtype=torch.float64, device=dev)
    s = timed(lambda: g.fill_f64(f64))
    bd = fill_breakdown(g, lambda: g.fill_f64(f64))
    out["c2_L8_2p28_f64"] = {"value": n / s, "unit": "float64/s", "ms": s * 1e3, "gbs": n * 8 / s / 1e9,
                             "roofline": stated(hbm(n * 8, s), bd,
                                                "generation kernel: 8-byte elements, one double per word "
                                                "(I2F.F64 + DMUL per word, 148 chunks, 4 warps per SM), beside the "
                                                "co-resident positioning GEMM of 1184 lane states",
                                                "positioning GEMM (148 chunks x 8 lanes = 1184 rows per fill)")}
    del f64
    # c3: 1024 generators (L=16, seeds 1..1024, full period) x 2^20 words, generator-major,
    # including the 1024 x 15 de-phasing jumps
    n = 1 << 20
    b3 = torch.empty(1024 * n, dtype=torch.uint32, device=dev)
    s = timed(lambda: V.batch_fill_u32(b3, 1, 1024, 16, n), reps=2)
    # the same call without generation (n_per_gen = 0: seeding + de-phasing only)
    tc = timed(lambda: V.batch_fill_u32(b3, 1, 1024, 16, 0), reps=2)
    r3 = hbm(1024 * n * 4, s)
    r3.update(breakdown_ms={"seed_and_dephase": tc * 1e3, "generation": (s - tc) * 1e3},
              limited_by="de-phasing: log2(16) = 4 FP4 tcgen05 GEMMs over 1024 x (1+2+4+8) lane states "
                         "(15360 rows x 19968^2 MACs) before 4 GiB of generation")
    out["c3_1024xL16_2p20_u32"] = {"value": 1024 * n / s, "unit": "uint32/s", "ms": s * 1e3, "roofline": r3,
                                   "note": "includes seeding + de-phasing of 15360 lane states (four FP4 GEMMs, matrices cached)"}
    del b3
    # c5: 4096 states (seeds 1..4096) jumped by 64-bit distances, then 624 outputs each
    seeds = np.arange(1, 4097, dtype=np.uint32)
    states = torch.from_numpy(V.seed_states(seeds).view(np.int32)).to(dev).view(torch.uint32)
    dists = np.random.default_rng(7).integers(0, 2**63, 4096, dtype=np.int64).view(np.uint64)
    jumped = torch.empty_like(states)
    s = timed(lambda: V.jump_states(states, dists, out=jumped), reps=2)
    out["c5_4096_jumps_64bit"] = {"value": 4096 / s, "unit": "state jumps/s", "ms": s * 1e3,
                                  "roofline": {"bound": "alu", "limited_by": "integer ALU issue of the polynomial "
                                               "jump (p(F)s as a word convolution: ~19960 coefficient steps x 20 "
                                               "words x LOP3 per jump); see profiles/r02_summary.md"},
                                  "note": "3 polynomial jumps per state from 16-bit digit tables (bits 16..63 of the 64-bit distance) + a direct advance by the low 16 bits"}
    # fused statistics consumer (monobit + chi2 byte histogram), 2^32 words, nothing stored
    n = 1 << 32
    g = V.VmtGenerator(5489, V.VmtConfig(32))
    s = timed(lambda: g.stat_counts(n), reps=2)
    out["stats_consumer_L32_2p32"] = {"value": n / s, "unit": "uint32/s", "ms": s * 1e3,
                                      "roofline": {"bound": "smem-atomic", "limited_by": "4 shared-memory atomics "
                                                   "per tempered word (byte histogram), ~0.31 warp-ATOMS per clock "
                                                   "per SM; nothing stored (DESIGN.md section 4.5)"}}
    # full-period jump matrix F^(2^19932) (the reference needs ~50 h of squarings)
    rows = torch.empty((19937, 312), dtype=torch.uint64, device=dev)
    s = timed(lambda: V.jump_matrix_pow2(19932, out=rows), reps=2)
    out["jump_matrix_2p19932"] = {"value": s * 1e3, "unit": "ms", "note": "19937 basis-state polynomial jumps",
                                  "roofline": {"bound": "alu", "limited_by": "the polynomial jump kernel "
                                               "(19937 jobs), as c5"}}
    return out


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    words = args.words
    vals = []
    for i in range(args.warmup + args.steps):
        v, s, x, done = reference_cpu(words, threads)
        if i >= args.warmup:
            vals.append((v, s))
    value = statistics.median(v for v, _ in vals)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": statistics.median(s for _, s in vals) * 1e3, "higher_is_better": True,
        "scaling": args.scaling, "vs_baseline": None, "dtype": "u32", "data": "synthetic (seeded generator)",
        "config": {"workload": "c4: L=32 VMT19937 stream, 2^34 uint32 per step", "total_words": words,
                   "reference_lanes": 16, "reference_jump_exponent": 16,
                   "note": "reference engine supports L<=16 (engine.hpp:43); M=16 AVX-512 engines, q=16 "
                           "(throughput is independent of q; full-period matrices take ~50 h)"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "reference",
                         "sample": f"{words} uint32 per step, {threads} threads x VmtEngine<16>::next_block_state "
                                   f"into DRAM ({cpu_model()})", "simd": reference_simd()},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# -------------------------------------------------------------------- ours --
def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2309_16682_b200 as V
    from paper_2309_16682_b200.dist import combine_xor, max_over_ranks, partition

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # VMT_BENCH_SHARED_GPU=1: harness test only -- every rank on cuda:0 with
    # gloo collectives (exercises the N>1 code path on a one-GPU box; its
    # numbers are not scaling measurements)
    shared = os.environ.get("VMT_BENCH_SHARED_GPU") == "1"
    if shared:
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if shared:
            dist.init_process_group("gloo")
        else:
            # communicator / nranks lines on stderr (the JSON line is on stdout)
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            dist.init_process_group("nccl", device_id=dev)
    coll = torch.device("cpu") if shared else dev  # device of the collectives' tensors
    # T = words the whole job generates per step (all ranks)
    T = args.words * world if args.scaling == "weak" else args.words
    start, count = partition(T, world, rank)

    torch.cuda.synchronize(dev)
    t_setup = time.perf_counter()
    g = V.VmtGenerator(SEED, V.VmtConfig(LANES), device=local)  # seed + full-period de-phasing
    setup_ms = (time.perf_counter() - t_setup) * 1e3
    g.set_tuning(max_chunks=args.chunks, variant=args.variant)
    g.set_prefetch(args.prefetch)
    out = torch.empty(count, dtype=torch.uint32, device=dev)
    stream = torch.cuda.current_stream(dev)

    def step():
        if args.mode == "store":
            g.fill_u32(out)
        else:
            g.checksum_xor(count, stream=stream.cuda_stream or 1)
        g.skip(T - count)  # the other ranks' share of this step

    # the clock/power poller starts before the warm-up, so the timed steps
    # follow the warm-up steps without an idle gap (the board's power state
    # is that of continuous load)
    clocks = ClockSampler(dev)
    g.seek(start)
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)

    g.set_profiling(True)  # CUDA events around each step's jump and generation launches
    g.profile_totals()
    clocks.start()
    s0 = g.stats()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        step()
    e1.record(stream)
    e1.synchronize()
    clocks.mark_end()
    s1 = g.stats()
    fills, jump_tot, gen_tot = g.profile_totals()
    g.set_profiling(False)

    # -- the same number of steps with the other positioning mode (serial GEMM
    # <-> co-resident GEMM), run straight after the timed steps so the board
    # is in the same (power-capped) state; reported beside the timed mode
    other_pf = 2 if args.prefetch == 0 else 0
    serial = None
    if args.mode == "store" and not args.no_extras:
        g.set_prefetch(other_pf)
        for _ in range(2):
            step()
        g.set_profiling(True)
        g.profile_totals()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record(stream)
        for _ in range(args.steps):
            step()
        f1.record(stream)
        f1.synchronize()
        sf, sj, sg = g.profile_totals()
        g.set_profiling(False)
        g.set_prefetch(args.prefetch)
        serial = {"prefetch": other_pf, "steps": args.steps, "ms_per_step": f0.elapsed_time(f1) / args.steps,
                  "gen_kernel": sg / max(sf, 1), "positioning": sj / max(sf, 1),
                  "gen_roofline_frac": count * 4 / (sg / max(sf, 1) * 1e-3) / 1e9 / measured_peak()[0],
                  "note": ("the tcgen05 FP4 positioning GEMM co-resident with the generation kernel "
                           "(vmt_set_prefetch(2), the library default): its cost moves inside gen_kernel"
                           if other_pf == 2 else
                           "vmt_set_prefetch(OFF): the tcgen05 FP4 positioning GEMM between the steps") +
                          "; run straight after the timed steps (2 more warm-up steps)"}
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    clk = clocks.stop()
    ms = e0.elapsed_time(e1) / args.steps
    ms = max_over_ranks(ms, coll)
    launches = sum(s1[k] - s0[k] for k in ("gen_launches", "jump_launches", "other_launches"))
    # the generation kernel's own duration and the positioning before it,
    # from the same timed steps
    gen_ms = max_over_ranks(gen_tot / max(fills, 1), coll)
    jump_ms = max_over_ranks(jump_tot / max(fills, 1), coll)

    # -- global checksum of one full 2^34 range (config 4 verification)
    g.seek(start)
    csum = combine_xor(g.checksum_xor(count), coll)
    torch.cuda.synchronize(dev)

    # -- end to end, fused consumer: the step's result is the 4-byte XOR
    # checksum read back to the host (config 4's no-store mode)
    g.seek(start)
    for _ in range(args.warmup):  # same warm-up as the timed store steps
        g.checksum_xor(count)
        g.skip(T - count)
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        g.checksum_xor(count)
        g.skip(T - count)
    xs = max_over_ranks((time.perf_counter() - t0) / args.steps, coll)
    e2e_xor = {"value": T / xs, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 4 * world,
               "ms_per_step": xs * 1e3, "mode": "fused XOR checksum, nothing stored",
               "note": "temper-free algebraic path: the kernel XORs the untempered words and tempers the "
                       "fold once (temper is GF(2)-linear) -- valid for this consumer only; the general "
                       "fused consumer that tempers every word is other_configs.stats_consumer_L32_2p32"}

    # -- end to end into pinned host memory through the public API
    e2e = None
    out = None  # the 64 GiB device buffer is no longer needed
    torch.cuda.empty_cache()
    # (N > 1: 2^32 words = 16 GiB of pinned host memory per rank instead of
    # the full 64 GiB share, so 8 ranks pin 128 GiB rather than 512 GiB; the
    # number is PCIe-bound and does not depend on the size past a few GiB)
    ew = count if world == 1 else min(count, 1 << 32)
    # never pin more than half of the host's available memory across the
    # node's ranks (one node: every rank of the job shares this host)
    try:
        import psutil
        avail_words = psutil.virtual_memory().available // 2 // world // 4
        ew = min(ew, max(avail_words >> 24 << 24, 0))
    except Exception:
        pass
    Te = ew * world
    if not args.no_e2e and args.mode == "store" and ew < (1 << 26):
        e2e = {"unavailable": f"host memory too small for a pinned end-to-end buffer per rank ({ew} words)"}
    elif not args.no_e2e and args.mode == "store":
        host, kind = None, None
        try:
            host = torch.empty(ew, dtype=torch.uint32, pin_memory=True)
            kind = "pinned"
        except Exception:
            if world == 1:
                host = np.empty(ew, np.uint32)
                kind = "pageable"
        ok = torch.tensor([1 if host is not None else 0], device=coll)
        if world > 1:
            dist.all_reduce(ok, op=dist.ReduceOp.MIN)
        if int(ok.item()) == 0:
            e2e = {"unavailable": "no pinned host memory for the end-to-end buffer on some rank"}
        else:
            g.set_prefetch(2)  # the public API's default positioning (co-resident prefetch)
            g.seek(rank * ew)
            g.fill_u32(host)  # warm-up
            g.skip(Te - ew)
            if world > 1:
                dist.barrier()
            t0 = time.perf_counter()
            for _ in range(args.e2e_steps):
                g.fill_u32(host)
                g.skip(Te - ew)
            e2e_s = (time.perf_counter() - t0) / args.e2e_steps
            e2e_s = max_over_ranks(e2e_s, coll)
            e2e = {"value": Te / e2e_s, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": Te * 4,
                   "ms_per_step": e2e_s * 1e3, "host_buffer": kind, "steps": args.e2e_steps,
                   "words_per_rank": ew}
        # the link the e2e number is bound by: a plain 1 GiB pinned D2H copy
        if kind == "pinned" and "value" in e2e:
            src = torch.empty(1 << 28, dtype=torch.uint32, device=dev)
            best = 0.0
            for _ in range(3):
                torch.cuda.synchronize()
                t1 = time.perf_counter()
                host[: 1 << 28].copy_(src, non_blocking=True)
                torch.cuda.synchronize()
                best = max(best, (1 << 30) / (time.perf_counter() - t1) / 1e9)
            # sustained: 16 back-to-back 1 GiB copies into distinct parts of the buffer
            parts = min(16, ew >> 28)
            torch.cuda.synchronize()
            t1 = time.perf_counter()
            for k in range(parts):
                host[k << 28: (k + 1) << 28].copy_(src, non_blocking=True)
            torch.cuda.synchronize()
            sustained = parts * (1 << 30) / (time.perf_counter() - t1) / 1e9 if parts else None
            e2e_gbs = Te * 4 / e2e_s / 1e9 / world
            e2e["link_probe"] = {"d2h_memcpy_gbs": best, "d2h_memcpy_sustained_gbs": sustained,
                                 "e2e_gbs": e2e_gbs, "frac": e2e_gbs / best,
                                 "frac_of_sustained": e2e_gbs / sustained if sustained else None,
                                 "note": "pinned cudaMemcpy D2H (PCIe), one 1 GiB copy (best of 3) and 16 "
                                         "back to back: the e2e fill moves 4 B per word over the same link"}
            del src
        del host

    # every rank's own step time, clocks and throughput (rank 0 prints them)
    mine = {"rank": rank, "device": local, "ms_per_step_local": e0.elapsed_time(e1) / args.steps,
            "gen_kernel_ms": gen_tot / max(fills, 1), "per_gpu_value": count / (e0.elapsed_time(e1) / args.steps * 1e-3),
            "sm_mhz": clk.get("sm_mhz") if isinstance(clk, dict) else None,
            "reasons": clk.get("reasons") if isinstance(clk, dict) else None}
    if world > 1:
        per_rank = [None] * world
        dist.all_gather_object(per_rank, mine)
    else:
        per_rank = [mine]

    peak, peak_src = measured_peak()
    # second denominator: pure-store probes over the same 64 GiB (after the
    # bench's own buffers are released)
    store_peaks = {}
    try:
        store_peaks = {"grid_stride_gbs": V.store_bandwidth(count * 4, 0, 2, local),
                       "chunk_per_cta_gbs": V.store_bandwidth(count * 4, 1, 1, local),
                       # random words, like the generator's output: the HBM interface power of
                       # the store stream alone approaches the board's 1000 W limit (DESIGN 4.1)
                       "chunk_per_cta_random_gbs": V.store_bandwidth(count * 4, 2, 1, local)}
    except Exception as e:
        store_peaks = {"error": str(e)}
    bytes_per_launch = count * 4
    achieved = bytes_per_launch / (gen_ms * 1e-3) / 1e9
    traffic = profiled_traffic()
    line = {
        "metric": METRIC, "value": T / (ms * 1e-3), "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": args.scaling,
        "vs_baseline": None, "dtype": "u32", "data": "synthetic (seeded generator, no inputs)",
        "config": {"workload": "c4: one L=32 VMT19937 stream, seed 5489, default full-period de-phasing "
                               "(q=19932), 2^34 uint32 per rank per step (weak) / per step (strong), "
                               "contiguous per-rank ranges",
                   "total_words": T, "lanes": LANES, "jump_exponent": g.jump_exponent(), "mode": args.mode,
                   "per_rank_words": count, "l2": "output >= 8 GiB per rank per step >> 126 MB L2 (no flush)",
                   "parallelism": f"stream partition x{world} ({args.scaling})"},
        "gpu_launches": launches,
        "per_gpu_value": count / (ms * 1e-3),
        "per_rank": per_rank,
        "timing_breakdown_ms": {"gen_kernel": gen_ms, "positioning": jump_ms, "setup_create": setup_ms,
                                "positioning_gemms": g.positioning_stats()["gemm_positionings"],
                                "prefetch": g.prefetch_stats(),
                                "positioning_mode": args.prefetch,
                                "other_positioning_mode": serial,
                                "note": "CUDA events on the fill's stream around the chunk positioning and the "
                                        "generation launch of every timed step. " + (
                                            "Steady state: each step's 4736 chunk lane states are one tcgen05 FP4 "
                                            "GEMM (vmt_posmma2_kernel, 4736 x 19968^2, ~0.75 ms) launched before "
                                            "the step's generation kernel ('positioning')"
                                            if args.prefetch == 0 else
                                            "Steady state: the next step's 4736 chunk lane states are computed "
                                            "during this step's generation kernel by the co-resident tcgen05 FP4 "
                                            "GEMM, so 'positioning' is only the wait for it and its cost shows up "
                                            "inside gen_kernel") + "; first steps: polynomial jumps, then the GEMM "
                                        "once the positioning matrix of the repeating step is built"},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": (traffic or {}).get("dram_bytes_per_launch"),
                     "kernel": "vmt_gen_kernel", "peak_source": peak_src,
                     "algorithmic_bytes_per_launch": bytes_per_launch,
                     "store_probe": dict(store_peaks, frac_of_grid_stride=(
                         achieved / store_peaks["grid_stride_gbs"] if "grid_stride_gbs" in store_peaks else None)),
                     "limited_by": (
                         "board power limit (sw_power_cap during the timed steps): storing random words at "
                         "~6.4 TB/s alone draws ~990 W of the 1000 W limit and twist + temper add ~210 pJ/word, so "
                         "the SM clock is lowered until both fit (profiles/r02_summary.md)"
                         if "sw_power_cap" in (clk.get("reasons") or []) else
                         "ALU issue at full clock (twist + temper: 9 ALU-pipe ops per word, ALU pipe ~79%) beside "
                         "the 64-bit output stores; DRAM traffic = the algorithmic bytes (roofline.traffic)")},
        "checksum_xor": f"0x{csum:08x}",
        "checksum_oracle": oracle_checksum(T, world, args),
        "clocks": clk,
        "e2e": e2e,
        "e2e_xor": e2e_xor,
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            threads = os.cpu_count() or 1
            v, s, x, done = reference_cpu(1 << 32, threads)
            line["cpu_baseline"] = {"value": v, "unit": UNIT, "cores": threads, "kind": "reference",
                                    "sample": f"{done} uint32 (2^32), {threads} threads x VmtEngine<16> "
                                              f"next_block_state into DRAM, q=16 ({cpu_model()}); "
                                              "L=32 unsupported by the reference",
                                    "simd": reference_simd()}
        except Exception as e:  # the reference build is optional on the box
            line["cpu_baseline"] = {"value": None, "unit": UNIT, "cores": 0, "kind": "reference",
                                    "sample": f"unavailable: {e}"}
    if rank == 0 and world == 1 and not args.no_extras:
        try:
            line["other_configs"] = extras(dev)
        except Exception as e:
            line["other_configs"] = {"error": f"{type(e).__name__}: {e}"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
