"""Summarise an ncu --set full report (.ncu-rep) into markdown: key throughput metrics, stalls, DRAM bytes."""
import csv
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe active %"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe active %"),
    ("SM_C.TriageCompute.smsp__pipe_tensor_subpipe_dmma_cycles_active.avg", "DMMA subpipe active cycles / SMSP"),
    ("TPC.TriageCompute.sm__pipe_tensor_subpipe_hmma_cycles_active_realtime.avg", "HMMA (tf32) subpipe active cycles / SM"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 throughput % of peak"),
    ("lts__t_bytes.sum", "L2 bytes"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_elapsed", "L1/shared-memory throughput % of peak"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "shared-memory wavefronts"),
    ("smsp__inst_executed.sum", "warp instructions executed"),
    ("sm__cycles_active.avg", "SM active cycles (avg)"),
    ("sm__cycles_active.max", "SM active cycles (max)"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "shared-memory bank conflicts"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__shared_mem_per_block_dynamic", "dyn smem/block"),
]


def main(path, out):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    h, u = rows[0], rows[1]
    lines = [f"# ncu summary: `{path.split('/')[-1]}`\n"]
    for r in rows[2:]:
        lines.append(f"## {r[h.index('Kernel Name')][:110]}\n")
        lines.append("| metric | value |\n|---|---|")
        for k, label in KEYS:
            if k in h:
                lines.append(f"| {label} (`{k}`) | {r[h.index(k)]} {u[h.index(k)]} |")
        st = []
        for i, name in enumerate(h):
            if name.startswith("smsp__pcsamp_warps_issue_stalled") and not name.endswith("not_issued"):
                try:
                    st.append((float(r[i].replace(",", "")), name[len("smsp__pcsamp_warps_issue_stalled_"):]))
                except ValueError:
                    pass
        tot = sum(v for v, _ in st) or 1.0
        lines.append("\nTop stall reasons (pc sampling): " +
                     ", ".join(f"{n} {100 * v / tot:.0f}%" for v, n in sorted(st, reverse=True)[:5]) + "\n")
    open(out, "w").write("\n".join(lines) + "\n")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
