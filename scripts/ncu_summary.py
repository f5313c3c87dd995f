# SPDX-License-Identifier: Apache-2.0
"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) and a
`--set full` report into markdown for profiles/.

  python scripts/ncu_summary.py LAUNCHES.csv [REPORT.ncu-rep] > profiles/rNN_*.md
"""
import collections
import csv
import subprocess
import sys


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr, agg = None, collections.OrderedDict()
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr is None or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = d["Kernel Name"].split("(")[0].replace("void ", "").replace("hg::", "")
        v = float(d["Metric Value"].replace(",", ""))
        v = {"nsecond": v / 1e3, "usecond": v, "msecond": v * 1e3}.get(d["Metric Unit"], v)
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += v
    # bench.py's roofline-denominator probes and the target's input upload (host-packed chunks
    # widened on the device, raw share narrowed) are not part of the step: listed, not shared
    upload = ("k_unpack24", "k_narrow")
    side = lambda k: "probe" in k or any(u in k for u in upload)
    tot = sum(v[1] for k, v in agg.items() if not side(k))
    out = ["| kernel | launches | total (ncu units) | share of the step's kernels |", "|---|---:|---:|---:|"]
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
        share = "(peak probe)" if "probe" in k else ("(input upload)" if side(k) else f"{v[1] / tot:.3f}")
        out.append(f"| {k} | {v[0]} | {v[1]:.1f} | {share} |")
    return "\n".join(out)


FIELDS = [
    ("gpu__time_duration.sum", "time"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM % peak"),
    ("launch__registers_per_thread", "regs/thread"),
    ("sm__warps_active.avg.per_cycle_active", "warps/SM"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA-pipe (IMAD) %"),
    ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "ALU-pipe %"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem bank conflicts"),
]


def full(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr, units = rows[0], rows[1]
    stall = [i for i, h in enumerate(hdr)
             if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio")]
    out = []
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")]
        out.append(f"### {name}\n")
        out.append("| metric | value |\n|---|---:|")
        for key, label in FIELDS:
            if key in hdr:
                i = hdr.index(key)
                out.append(f"| {label} (`{key}`) | {r[i]} {units[i]} |")
        st = sorted(((float(r[i] or 0), hdr[i][34:-23]) for i in stall), reverse=True)[:5]
        out.append("| top stalls (per issue) | " + ", ".join(f"{n} {v:.2f}" for v, n in st) + " |\n")
    return "\n".join(out)


if __name__ == "__main__":
    print("## Launch list (cold-cache, serialised; compare shares)\n")
    print(launches(sys.argv[1]))
    if len(sys.argv) > 2:
        print("\n## `ncu --set full` per kernel\n")
        print(full(sys.argv[2]))
