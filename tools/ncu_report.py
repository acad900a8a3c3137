"""Condense an ncu --set full report (.ncu-rep) into the metrics this project cites."""
import csv, subprocess, sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "dram__bytes_read.sum.per_second",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "lts__t_sector_hit_rate.pct",
    "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active", "launch__cluster_dim_x",
    "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_subpipe_imma_cycles_active_realtime.avg", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
]


def main(path, out=None):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr, units = rows[0], rows[1]
    lines = [f"# {path}"]
    seen = set()
    for vals in rows[2:]:
        name = vals[hdr.index('Kernel Name')]
        if name in seen:  # one block per distinct kernel (first launch)
            continue
        seen.add(name)
        lines += kernel_block(hdr, units, vals)
    text = "\n".join(lines) + "\n"
    if out:
        open(out, "w").write(text)
    print(text)


def kernel_block(hdr, units, vals):
    lines = ["", f"kernel: {vals[hdr.index('Kernel Name')]}"]
    for k in KEYS:
        if k in hdr:
            i = hdr.index(k)
            lines.append(f"{k} = {vals[i]} {units[i]}")
    stalls = []
    for h, v in zip(hdr, vals):
        if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued"):
            try:
                stalls.append((float(v.replace(",", "")), h.replace("smsp__pcsamp_warps_issue_stalled_", "")))
            except ValueError:
                pass
    tot = sum(v for v, _ in stalls) or 1.0
    lines.append("top stall reasons (pc sampling): " + ", ".join(f"{n} {v / tot:.0%}" for v, n in sorted(stalls, reverse=True)[:6]))
    return lines


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else None)
