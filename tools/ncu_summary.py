"""Summarise ncu captures for profiles/ (run in the build container).

    python tools/ncu_summary.py launches <launches.csv>            # per-kernel share of a launch list
    python tools/ncu_summary.py full <report.ncu-rep> [...]         # key --set full metrics per kernel
    python tools/ncu_summary.py traffic <report.ncu-rep> KERNEL=PHASE:ALG_BYTES ...
"""

from __future__ import annotations

import collections
import csv
import io
import json
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM % of peak"),
    ("lts__t_bytes.sum", "L2 bytes"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe active %"),
    ("sm__pipe_tensor_subpipe_imma_cycles_active.avg.pct_of_peak_sustained_active", "IMMA subpipe active %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem bank conflicts"),
]


def _raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def full(reps):
    lines = []
    for rep in reps:
        hdr, units, rows = _raw(rep)
        lines.append(f"### `{rep.split('/')[-1]}`\n")
        lines.append("| kernel | " + " | ".join(n for _, n in KEYS) + " |")
        lines.append("|" + "---|" * (len(KEYS) + 1))
        for r in rows:
            name = r[hdr.index("Kernel Name")].split("(")[0].replace("mmj::<unnamed>::", "").replace("mmj::", "")
            vals = []
            for k, _ in KEYS:
                if k in hdr:
                    i = hdr.index(k)
                    vals.append(f"{r[i]} {units[i]}".strip())
                else:
                    vals.append("-")
            lines.append(f"| {name[:40]} | " + " | ".join(vals) + " |")
        stalls = {}
        for r in rows:
            name = r[hdr.index("Kernel Name")].split("(")[0].split("::")[-1]
            st = {h.replace("smsp__pcsamp_warps_issue_stalled_", ""): int(float(r[i] or 0))
                  for i, h in enumerate(hdr)
                  if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued")}
            top = sorted(st.items(), key=lambda kv: -kv[1])[:5]
            stalls[name] = ", ".join(f"{k} {v}" for k, v in top)
        lines.append("\nTop warp-stall samples: " + "; ".join(f"**{k}**: {v}" for k, v in stalls.items()) + "\n")
    print("\n".join(lines))


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    hdr = rows[hi]
    ki, vi, mi = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Name")
    tot, cnt = collections.Counter(), collections.Counter()
    for r in rows[hi + 1:]:
        if len(r) > vi and r[mi] == "gpu__time_duration.sum":
            name = r[ki].split("(")[0]
            tot[name] += float(r[vi])
            cnt[name] += 1
    s = sum(tot.values())
    print("| kernel | launches | total us | share |\n|---|---|---|---|")
    for k, v in tot.most_common():
        print(f"| {k[:70]} | {cnt[k]} | {v / 1e3:.1f} | {100 * v / s:.1f}% |")


def traffic(rep, specs):
    hdr, units, rows = _raw(rep)
    out = {}
    for spec in specs:
        kern, rest = spec.split("=")
        phase, alg = rest.split(":")
        for r in rows:
            if kern in r[hdr.index("Kernel Name")]:
                rd = float(r[hdr.index("dram__bytes_read.sum")])
                wr = float(r[hdr.index("dram__bytes_write.sum")])
                scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
                rd *= scale.get(units[hdr.index("dram__bytes_read.sum")], 1)
                wr *= scale.get(units[hdr.index("dram__bytes_write.sum")], 1)
                out[phase] = {"kernel": kern, "dram_bytes_per_launch": rd + wr, "dram_read": rd, "dram_write": wr,
                              "algorithmic_bytes_per_launch": float(alg), "traffic_over_algorithmic": (rd + wr) / float(alg),
                              "source": rep.split("/")[-1]}
                break
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    cmd = sys.argv[1]
    if cmd == "full":
        full(sys.argv[2:])
    elif cmd == "launches":
        launches(sys.argv[2])
    elif cmd == "traffic":
        traffic(sys.argv[2], sys.argv[3:])
