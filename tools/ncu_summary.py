"""Summarise ncu --set full reports: time, DRAM bytes, L2/DRAM/tensor utilisation per kernel."""
import csv, io, subprocess, sys
WANT = [("gpu__time_duration.sum", "us", 1e-3), ("dram__bytes_read.sum", "MB_rd", 1.0), ("dram__bytes_write.sum", "MB_wr", 1.0),
        ("lts__t_bytes.sum", "L2_MB", 1.0),
        ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram%", 1), ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "l2%", 1),
        ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor%", 1),
        ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "lsu%", 1),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "occ%", 1), ("launch__registers_per_thread", "regs", 1)]
for rep in sys.argv[1:]:
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    idx = {h: i for i, h in enumerate(hdr)}
    for d in rows[2:]:
        parts = [d[idx["Kernel Name"]][:34]]
        for m, lab, sc in WANT:
            if m in idx:
                try:
                    v = float(d[idx[m]].replace(",", ""))
                    u = units[idx[m]]
                    if lab.startswith("MB") or lab == "L2_MB":
                        v = v * {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}.get(u, 1.0)
                    elif lab == "us":
                        v = v * {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3}.get(u, 1.0)
                    parts.append(f"{lab}={v:.1f}")
                except ValueError:
                    pass
        print(" ".join(parts))
