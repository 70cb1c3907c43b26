"""Summarise ncu exports committed under profiles/ (run here, no GPU needed).

    python profiles/summarize.py r01 profiles/r01_ncu_full_raw.csv profiles/r01_launches_text_like.csv

writes profiles/<round>_summary.md and profiles/ncu_traffic.json (per-launch
DRAM bytes of the step's kernels, which bench.py reports as roofline.traffic).
"""
import csv
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
METRICS = [
    ("gpu__time_duration.sum", "time"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM %"),
    ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "ALU pipe %"),
    ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "L1TEX %"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 %"),
    ("launch__registers_per_thread", "regs"),
]
# bench.py phase -> kernel whose launch dominates it, and the grid of the collection-size launch
PHASE_KERNEL = {"build_minwise": "minwise_kernel", "build_oph_hoph": "build_kernel", "compare_full": "probe_kernel"}


def to_bytes(v, unit):
    v = float(v)
    return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)


def raw_rows(path):
    rows = list(csv.reader(open(path)))
    hdr, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        d = {}
        for key, _ in METRICS + [("Kernel Name", ""), ("Grid Size", "")]:
            if key in hdr:
                i = hdr.index(key)
                d[key] = (r[i], units[i])
        out.append(d)
    return out


def launches(path):
    lines = open(path).read().splitlines()
    start = [i for i, l in enumerate(lines) if l.startswith('"ID"')][0]
    return list(csv.DictReader(lines[start:]))


def main(rnd, raw, lau):
    md = [f"# {rnd}: ncu summaries (B200, sm_100a)\n"]
    md.append(f"Source: `{os.path.basename(raw)}` (`ncu --set full --clock-control none`), "
              f"`{os.path.basename(lau)}` (`ncu --metrics gpu__time_duration.sum`, cold-cache, serialised).\n")
    md.append("## Kernels (ncu --set full)\n")
    md.append("| kernel | grid | " + " | ".join(n for _, n in METRICS) + " |")
    md.append("|---" * (len(METRICS) + 2) + "|")
    traffic = {}
    for d in raw_rows(raw):
        name = d["Kernel Name"][0].split("(")[0].replace("void ", "")
        cells = []
        for key, _ in METRICS:
            v, u = d.get(key, ("", ""))
            cells.append(f"{v} {u}".strip())
        md.append(f"| {name} | {d['Grid Size'][0]} | " + " | ".join(cells) + " |")
        if "dram__bytes_read.sum" in d:
            rb = to_bytes(*d["dram__bytes_read.sum"]) + to_bytes(*d["dram__bytes_write.sum"])
            for phase, kern in PHASE_KERNEL.items():
                big = d["Grid Size"][0].split(",")[0].strip("( ")
                if kern in name and int(big) > 500:
                    traffic.setdefault(phase, rb)
    rows = launches(lau)
    tot = {}
    for r in rows:
        n = r["Kernel Name"].split("(")[0].replace("void ", "").replace("ophgpu::", "")
        tot[n] = tot.get(n, 0.0) + float(r["Metric Value"]) / 1e3
    all_us = sum(tot.values())
    md.append("\n## Launch list: device time by kernel over the whole captured run\n")
    md.append("| kernel | total us | share |")
    md.append("|---|---|---|")
    for n, t in sorted(tot.items(), key=lambda x: -x[1]):
        md.append(f"| {n} | {t:.1f} | {100 * t / all_us:.1f}% |")
    with open(os.path.join(HERE, f"{rnd}_summary.md"), "w") as f:
        f.write("\n".join(md) + "\n")
    with open(os.path.join(HERE, "ncu_traffic.json"), "w") as f:
        json.dump(traffic, f, indent=1)
    print("\n".join(md))
    print(traffic)


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3])
