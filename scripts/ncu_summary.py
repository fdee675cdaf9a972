"""Summarise ncu reports (run here, no GPU): per kernel the duration, DRAM
bytes, pipe utilisation and top stall reasons -> markdown on stdout.
  python scripts/ncu_summary.py gpurun_out/r01_shortlist_pair.ncu-rep ..."""
import csv, subprocess, sys

KEYS = [("gpu__time_duration.sum", "duration"), ("dram__bytes_read.sum", "DRAM read"),
        ("dram__bytes_write.sum", "DRAM write"),
        ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
        ("sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed", "tensor pipe active %"),
        ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
        ("lts__t_sector_hit_rate.pct", "L2 hit %"), ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
        ("launch__registers_per_thread", "regs/thread"), ("launch__grid_size", "grid"), ("launch__block_size", "block")]
STALLS = ["long_scoreboard", "wait", "barrier", "short_scoreboard", "math_pipe_throttle", "mio_throttle",
          "lg_throttle", "no_instruction", "branch_resolving", "membar", "sleeping", "selected"]
for rep in sys.argv[1:]:
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, u = rows[0], rows[1]
    print(f"### `{rep.split('/')[-1]}`\n")
    seen = set()
    for r in rows[2:]:
        name = r[h.index("Kernel Name")].split("(")[0]
        if name in seen:
            continue
        seen.add(name)
        print(f"**{name}**\n")
        for k, label in KEYS:
            if k in h:
                i = h.index(k)
                print(f"- {label}: {r[i]} {u[i]}")
        st = []
        for sname in STALLS:
            k = f"smsp__average_warps_issue_stalled_{sname}_per_issue_active.ratio"
            if k in h and r[h.index(k)] not in ("", "0"):
                st.append((float(r[h.index(k)]), sname))
        st.sort(reverse=True)
        print("- top stalls (warps per issue): " + ", ".join(f"{n} {v:.2f}" for v, n in st[:4]) + "\n")
