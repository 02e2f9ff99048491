"""Key counters of every launch in an `ncu --set full` report:
python tools/ncu_rep.py report.ncu-rep [...]"""
import csv
import io
import subprocess
import sys

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("sm__inst_issued.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum", "smem load wavefronts"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "smem load bank conflicts"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum", "smem store wavefronts"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum", "smem store bank conflicts"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram throughput %"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "l1tex throughput %"),
    ("sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe %"),
]


def _bytes(v, unit):
    return float(v) * {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0}.get(unit, 1.0)


def summarize(rep, metrics=METRICS):
    """(text lines, DRAM bytes per launch) of every launch in `rep`."""
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    idx = {h: i for i, h in enumerate(hdr)}
    out, traffic = [], []
    for n, r in enumerate(rows[2:]):
        out.append(f"launch {n}: {r[idx['Kernel Name']]}  grid {r[idx.get('launch__grid_size', 0)]}")
        for key, label in metrics:
            if key in idx:
                out.append(f"  {label:28s} {r[idx[key]]:>16s} {units[idx[key]]}")
        st = {h: float(r[i]) for h, i in idx.items()
              if h.startswith("smsp__pcsamp_warps_issue_stalled") and not h.endswith("not_issued") and r[i]}
        tot = sum(st.values()) or 1.0
        out.append("  stall samples: " + ", ".join(
            f"{k.replace('smsp__pcsamp_warps_issue_stalled_', '')} {v / tot * 100:.0f}%"
            for k, v in sorted(st.items(), key=lambda kv: -kv[1])[:8]))
        rd = _bytes(r[idx["dram__bytes_read.sum"]], units[idx["dram__bytes_read.sum"]])
        wr = _bytes(r[idx["dram__bytes_write.sum"]], units[idx["dram__bytes_write.sum"]])
        traffic.append(rd + wr)
        out.append("")
    return out, traffic


if __name__ == "__main__":
    for rep in sys.argv[1:]:
        print("==", rep)
        print("\n".join(summarize(rep)[0]))
