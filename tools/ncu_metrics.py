"""Print the key raw metrics of every kernel in an ncu report (development tool)."""
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "smsp__inst_executed.sum", "sm__cycles_elapsed.avg.per_second", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed.sum", "smsp__warps_active.avg.per_cycle_active", "smsp__warps_eligible.avg.per_cycle_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "launch__registers_per_thread", "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts.sum.pct_of_peak_sustained_elapsed", "launch__grid_size", "launch__block_size"]
STALLS = "smsp__pcsamp_warps_issue_stalled_"


def main(path, n=None):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[0]
    for row in rows[2:]:
        d = dict(zip(hdr, row))
        print("==", d.get("Kernel Name", "")[:90])
        for k in KEYS:
            if k in d:
                print(f"  {k:70s} {d[k]}")
        if n:
            inst = float((d.get("sm__inst_executed.sum") or d["smsp__inst_executed.sum"]).replace(",", ""))
            print(f"  thread-instructions per element: {inst * 32 / n:.1f}")
            sh = float(d["l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"].replace(",", ""))
            print(f"  shared wavefronts per 32 elements: {sh * 32 / n:.1f}")
        st = {k[len(STALLS):]: float(v.replace(",", "")) for k, v in d.items()
              if k.startswith(STALLS) and not k.endswith("not_issued") and v not in ("", "0")}
        tot = sum(st.values()) or 1
        print("  stalls:", ", ".join(f"{k} {100 * v / tot:.0f}%" for k, v in sorted(st.items(), key=lambda x: -x[1])[:9]))


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else None)
