"""Summarize ncu output into the markdown kept under profiles/.

    python profiles/summarize.py launches <launches.csv>         # per-kernel share of a launch list
    python profiles/summarize.py report <file.ncu-rep> [regex]   # key metrics + stall reasons per launch

The launch list comes from
    ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file X.csv <cmd>
(cold-cache, serialised launches: compare shares, not absolutes), the report
from ncu --set full --clock-control none --import-source on -k regex:... -o X <cmd>.
"""
import collections
import csv
import io
import re
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration (us)"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe % (active)"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe % (active)"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue slots busy %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__occupancy_limit_registers", "CTA limit (regs)"),
    ("launch__occupancy_limit_shared_mem", "CTA limit (smem)"),
    ("dram__bytes_read.sum", "DRAM read (MB)"),
    ("dram__bytes_write.sum", "DRAM write (MB)"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput %"),
    ("lts__t_bytes.sum", "L2 traffic (MB)"),
    ("lts__t_sectors.sum", "L2 sectors (x32 B)"),
    ("TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
     "tensor pipe active % (elapsed)"),
    ("sm__ops_path_tensor_op_utchmma_src_tf32_dst_fp32_sparsity_off.sum.pct_of_peak_sustained_elapsed",
     "tcgen05 tf32 MMA ops % of peak"),
    ("sm__ops_path_tensor_op_utchmma_src_fp16_dst_fp32_sparsity_off.sum.pct_of_peak_sustained_elapsed",
     "tcgen05 f16 MMA ops % of peak"),
    ("sm__inst_executed_pipe_tmem.avg.pct_of_peak_sustained_active", "TMEM pipe inst % (active)"),
    ("sm__inst_executed_pipe_tensor_subpipe_hmma.avg.pct_of_peak_sustained_active", "legacy HMMA pipe % (active)"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", "smem LSU wavefronts % of peak"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
]


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[hdr + 1:]:
        if len(r) <= vi:
            continue
        try:
            v = float(r[vi].replace(",", ""))
        except ValueError:
            continue
        scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "nsecond": 1e-3, "ms": 1e3, "msecond": 1e3}.get(r[ui], 1e-3)
        name = re.sub(r"\(.*", "", r[ki]).replace("(anonymous namespace)::", "")
        agg[name][0] += 1
        agg[name][1] += v * scale
    tot = sum(v[1] for v in agg.values())
    print("| kernel | launches | total (ms) | avg (us) | share |")
    print("|---|---:|---:|---:|---:|")
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"| `{k}` | {v[0]} | {v[1] / 1e3:.3f} | {v[1] / v[0]:.1f} | {v[1] / tot:.3f} |")


def report(path, regex=None):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    h, units = r[0], r[1]
    seen = set()
    for v in r[2:]:
        name = v[h.index("Kernel Name")]
        if regex and not re.search(regex, name):
            continue
        short = re.sub(r"[(].*", "", name)
        if short in seen:  # one launch per kernel
            continue
        seen.add(short)
        print(f"### `{re.sub(r'[(].*', '', name)}`\n")
        print("| metric | value |")
        print("|---|---:|")
        for key, label in KEYS:
            if key not in h:
                continue
            x = v[h.index(key)]
            unit = units[h.index(key)]
            try:
                f = float(x.replace(",", ""))
                if key.endswith("bytes.sum") or key.endswith("bytes_read.sum") or key.endswith("bytes_write.sum"):
                    f = f * {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}.get(unit, 1.0)
                if key == "gpu__time_duration.sum":
                    f = f * {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(unit, 1.0)
                x = f"{f:.2f}"
            except ValueError:
                pass
            print(f"| {label} | {x} |")
        try:  # achieved DRAM bandwidth of the launch (cold-cache replay)
            def mb(key):
                f = float(v[h.index(key)].replace(",", ""))
                return f * {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}.get(units[h.index(key)], 1.0)
            dur = float(v[h.index("gpu__time_duration.sum")].replace(",", "")) * {
                "nsecond": 1e-9, "ns": 1e-9, "usecond": 1e-6, "us": 1e-6, "msecond": 1e-3, "ms": 1e-3}.get(
                units[h.index("gpu__time_duration.sum")], 1e-9)
            print(f"| DRAM GB/s achieved (read+write / duration) | "
                  f"{(mb('dram__bytes_read.sum') + mb('dram__bytes_write.sum')) * 1e6 / dur / 1e9:.0f} |")
        except (ValueError, KeyError):
            pass
        st = [(n, v[i]) for i, n in enumerate(h)
              if n.startswith("smsp__average_warps_issue_stalled") and n.endswith("per_issue_active.ratio")]
        st = sorted(st, key=lambda a: -float(a[1] or 0))[:6]
        print("| top stalls (warps per issue) | " + ", ".join(
            f"{n.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', '')} "
            f"{float(x):.2f}" for n, x in st) + " |\n")


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2])
    else:
        report(sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else None)
