"""Development aid: one-screen summary of `ncu --page raw --csv` exports (profiles/)."""
import csv
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active", "DMMA pipe active %"),
    ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "FP64 (non-tensor) pipe %"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("launch__registers_per_thread", "registers / thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("smsp__inst_executed.sum", "instructions"),
    ("l1tex__t_bytes_pipe_lsu_mem_local_op_ld.sum", "local (spill) load bytes"),
    ("l1tex__t_bytes_pipe_lsu_mem_local_op_st.sum", "local (spill) store bytes"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem bank conflicts"),
]


def summarize(path):
    rows = list(csv.reader(open(path)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    ix = {h: i for i, h in enumerate(hdr)}
    out = [f"== {path}", f"   kernel: {vals[ix['Kernel Name']][:110]}"]
    for k, name in KEYS:
        if k in ix:
            out.append(f"   {name:28s} {vals[ix[k]]:>16s} {units[ix[k]]}")
    stalls = []
    for h, i in ix.items():
        if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("_not_issued"):
            try:
                stalls.append((float(vals[i]), h.replace("smsp__pcsamp_warps_issue_stalled_", "")))
            except ValueError:
                pass
    tot = sum(v for v, _ in stalls) or 1.0
    out.append("   stall samples (share): " + ", ".join(f"{n} {100 * v / tot:.1f}%" for v, n in sorted(stalls, reverse=True)[:6]))
    return "\n".join(out)


if __name__ == "__main__":
    print("\n".join(summarize(p) for p in sys.argv[1:]))
