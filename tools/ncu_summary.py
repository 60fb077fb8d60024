"""Summarise ncu artefacts into profiles/*.md.

  python tools/ncu_summary.py launches <launches.csv> <out.md>    # per-kernel device-time share
  python tools/ncu_summary.py kernel   <report.ncu-rep> <out.md>  # key --set full metrics of one kernel
  python tools/ncu_summary.py traffic  <report.ncu-rep> <out.json> <config>  # + DRAM bytes per launch
"""
import collections
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("dram__bytes_read.sum.pct_of_peak_sustained_elapsed", "DRAM read % of peak"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "ALU pipe %"),
    ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("sm__pipe_tensor_subpipe_imma_cycles_active.avg.pct_of_peak_sustained_active", "IMMA pipe % (legacy mma.sync)"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe active % (tcgen05)"),
    ("sm__ops_path_tensor_src_fp4_dst_fp32.sum", "FP4 tensor ops (2 x MAC)"),
    ("sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_active", "TMEM active %"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__block_size", "block size"),
    ("launch__grid_size", "grid size"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem bank conflicts"),
]


def launches(path, out):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[start]
    iN, iV, iU = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    iM = hdr.index("Metric Name")
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])  # launches, ns, DRAM bytes
    scale = {"nsecond": 1, "usecond": 1e3, "msecond": 1e6, "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    for r in rows[start + 1:]:
        if len(r) <= iV:
            continue
        name = r[iN].split("(")[0].replace("void ", "")
        v = float(r[iV].replace(",", "")) * scale.get(r[iU], 1)
        if r[iM] == "gpu__time_duration.sum":
            agg[name][0] += 1
            agg[name][1] += v
        elif r[iM].startswith("dram__bytes_"):
            agg[name][2] += v
    tot = sum(v[1] for v in agg.values())
    with open(out, "w") as f:
        f.write(f"# Launch list (`ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum "
                f"--clock-control none`), from `{path}`\n\n")
        f.write("Cold-cache, serialised per-launch times: compare shares, not absolutes.\n\n")
        f.write("| kernel | launches | total us | share | avg us | DRAM MB / launch |\n|---|---|---|---|---|---|\n")
        for k, (c, v, b) in sorted(agg.items(), key=lambda x: -x[1][1]):
            f.write(f"| `{k}` | {c} | {v / 1e3:.1f} | {100 * v / tot:.1f} % | {v / c / 1e3:.2f} | {b / c / 1e6:.1f} |\n")


def kernel(path, out):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    d = {h: (u, v) for h, u, v in zip(hdr, units, vals)}
    stalls = []
    for h, (u, v) in d.items():
        if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued"):
            try:
                stalls.append((float(v), h.replace("smsp__pcsamp_warps_issue_stalled_", "")))
            except ValueError:
                pass
    tot = sum(s for s, _ in stalls) or 1
    with open(out, "w") as f:
        f.write(f"# ncu --set full summary: `{d.get('Kernel Name', ('', '?'))[1]}`\n\nSource: `{path}`\n\n")
        f.write("| metric | value | unit |\n|---|---|---|\n")
        for key, label in KEYS:
            if key in d:
                f.write(f"| {label} (`{key}`) | {d[key][1]} | {d[key][0]} |\n")
        f.write("\n## Warp stall samples\n\n| reason | share |\n|---|---|\n")
        for s, n in sorted(stalls, reverse=True)[:10]:
            f.write(f"| {n} | {100 * s / tot:.1f} % |\n")
    return d


def traffic(path, out_json, config):
    """DRAM read + write per launch of the captured kernel -> bench.py's roofline `traffic`."""
    import json
    d = kernel(path, out_json.replace(".json", ".md"))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    b = sum(float(d[k][1].replace(",", "")) * scale[d[k][0]] for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
    name = d.get("Kernel Name", ("", "?"))[1]
    json.dump({"kernel": name.split("<")[0].replace("void ", "").split("::")[-1], "kernel_full": name,
               "dram_bytes_per_launch": b, "config": int(config), "source": path}, open(out_json, "w"), indent=1)


if __name__ == "__main__":
    {"launches": launches, "kernel": kernel, "traffic": traffic}[sys.argv[1]](*sys.argv[2:])
