"""Round-2 summaries of profiles/scripts/profile_r02.sh captures (run here,
with ncu on PATH, after the GPU call merged gpurun_out/). Usage:
  summarize_r02.py REPORT.ncu-rep [...]   markdown block per report
  summarize_r02.py --launches FILE.csv    launch-list shares"""
import collections
import csv
import io
import subprocess
import sys

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "ALU pipe %"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("sm__issue_active.avg.pct_of_peak_sustained_elapsed", "issue active %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("launch__registers_per_thread", "registers"),
    ("launch__shared_mem_per_block_dynamic", "dynamic shared memory per CTA"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem bank conflicts"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe %"),
]


def raw(rep, k=0):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    h, u, v = rows[0], rows[1], rows[2 + k]
    return {h[i]: (v[i], u[i]) for i in range(len(h))}, h, v


def stalls(h, v):
    st = [(h[i].replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""),
           float(v[i])) for i in range(len(h))
          if h[i].startswith("smsp__average_warps_issue_stalled") and h[i].endswith("per_issue_active.ratio")]
    return sorted([s for s in st if s[1] > 0.02], key=lambda t: -t[1])[:8]


def report(rep):
    m, h, v = raw(rep)
    print(f"\n### {rep.split('/')[-1]}: {m['Kernel Name'][0] if 'Kernel Name' in m else ''}")
    for key, label in METRICS:
        if key in m:
            print(f"- {label}: {m[key][0]} {m[key][1]}")
    print("- stalls per issue: " + ", ".join(f"{k} {x:.2f}" for k, x in stalls(h, v)))


def launches(path):
    rows = list(csv.reader(open(path)))
    i = [k for k, r in enumerate(rows) if r and r[0] == "ID"][0]
    hdr, data = rows[i], rows[i + 1:]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = collections.OrderedDict()
    for r in data:
        if len(r) <= vi:
            continue
        ms = float(r[vi].replace(",", "")) * {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "nsecond": 1e-6,
                                              "ms": 1, "msecond": 1}.get(r[ui], 1e-6)
        a = agg.setdefault(r[ki].split("(")[0], [0, 0.0])
        a[0] += 1
        a[1] += ms
    tot = sum(a[1] for a in agg.values())
    print(f"\n{path.split('/')[-1]}\n\n| kernel | launches | avg ms | share |\n|---|---|---|---|")
    for k, (c, t) in agg.items():
        print(f"| {k} | {c} | {t / c:.3f} | {100 * t / tot:.1f}% |")


if __name__ == "__main__":
    if sys.argv[1] == "--launches":
        for p in sys.argv[2:]:
            launches(p)
    else:
        for p in sys.argv[1:]:
            report(p)
