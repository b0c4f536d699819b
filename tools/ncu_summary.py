"""Summarise an ncu report (--set full) into markdown for profiles/: duration, DRAM traffic,
tensor-pipe / MUFU / FMA utilisation, registers, top stall reasons and top SASS lines."""
import csv
import io
import subprocess
import sys


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    units = dict(zip(rows[0], rows[1]))
    return [dict(zip(rows[0], r)) for r in rows[2:]], units


def sass_top(rep, k=12):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[1]
    data = rows[2:]
    iw = hdr.index("Warp Stall Sampling (All Samples)")
    isrc = hdr.index("Source")
    def num(r):
        try:
            return float(r[iw] or 0)
        except (ValueError, IndexError):  # repeated header rows of multi-kernel reports
            return 0.0
    tot = sum(num(r) for r in data) or 1.0
    top = sorted(data, key=lambda r: -num(r))[:k]
    return [(num(r) / tot * 100, r[isrc].strip()) for r in top]


def f(d, key, scale=1.0, fmt="{:.2f}"):
    v = d.get(key)
    try:
        return fmt.format(float(v) * scale)
    except (TypeError, ValueError):
        return "n/a"


def main(rep, title):
    recs, units = raw(rep)
    for d in recs:
        name = d.get("Kernel Name", "?")
        print(f"### {title}: `{name[:90]}`\n")
        print("| metric | value |\n|---|---|")
        print(f"| duration (ncu, cold/serialised) | {f(d, 'gpu__time_duration.sum', 1.0, '{:.3f}')} "
              f"{units.get('gpu__time_duration.sum', '')} |")
        print(f"| dram read + write per launch | {f(d, 'dram__bytes_read.sum')} "
              f"{units.get('dram__bytes_read.sum', '')} + {f(d, 'dram__bytes_write.sum')} "
              f"{units.get('dram__bytes_write.sum', '')} |")
        for key, lab in (("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor pipe active %"),
                         ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "XU (MUFU) pipe %"),
                         ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "FMA pipe %"),
                         ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "ALU pipe %"),
                         ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU pipe %"),
                         ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput %"),
                         ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
                         ("launch__registers_per_thread", "registers/thread")):
            print(f"| {lab} | {f(d, key)} |")
        stalls = sorted(((k.replace("smsp__pcsamp_warps_issue_stalled_", ""), float(v or 0)) for k, v in d.items()
                         if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")),
                        key=lambda x: -x[1])[:6]
        tot = sum(float(v or 0) for k, v in d.items() if k.startswith("smsp__pcsamp_warps_issue_stalled_")
                  and not k.endswith("not_issued")) or 1.0
        print(f"| top stall reasons (share of samples) | " +
              ", ".join(f"{k} {v / tot * 100:.0f}%" for k, v in stalls) + " |")
        print()
    print("Top SASS lines by stall samples:\n")
    print("```")
    for pct, src in sass_top(rep):
        print(f"{pct:5.1f}%  {src[:100]}")
    print("```\n")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else sys.argv[1])
