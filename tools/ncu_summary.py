"""One-page summary of an ncu --set full report (duration, DRAM traffic, throughput, tensor pipe, occupancy, stalls)."""
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram throughput % of peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    # tcgen05 (UMMA) utilisation on sm_100: the hmma sub-pipe's active cycles (the "bf16 tensor ops"
    # and instruction-count counters read ~0 for tcgen05.mma issued by one thread)
    ("sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_active", "UMMA (tcgen05) pipe active % (active cycles)"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor pipe active % (elapsed)"),
    ("l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", "smem read by tensor pipe % of peak"),
    ("sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active", "tc pipe cycles %"),
    ("lts__t_bytes.sum", "L2 bytes"),
    ("sm__warps_active.avg.per_cycle_active", "warps active / SM"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock (Hz)"),
]


def main(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    head, units = rows[0], rows[1]
    for r in rows[2:]:
        name = r[head.index("Kernel Name")][:90]
        print(f"== {name}")
        for key, label in KEYS:
            if key in head:
                i = head.index(key)
                print(f"   {label:34s} {r[i]} {units[i]}")
        stalls = []
        for i, n in enumerate(head):
            if n.startswith("smsp__pcsamp_warps_issue_stalled_") and not n.endswith("not_issued"):
                try:
                    stalls.append((float(r[i]), n.replace("smsp__pcsamp_warps_issue_stalled_", "")))
                except ValueError:
                    pass
        tot = sum(s for s, _ in stalls) or 1.0
        print("   top stalls: " + ", ".join(f"{n} {s / tot:.0%}" for s, n in sorted(stalls, reverse=True)[:5]))


if __name__ == "__main__":
    for p in sys.argv[1:]:
        main(p)
