"""Per-launch summary of an `ncu --page raw --csv` export (one row per profiled kernel).
usage: python tools/ncu_raw_summary.py RAW.csv [names...]"""
import csv, sys
WANT = [("gpu__time_duration.sum", "us"), ("dram__bytes_read.sum", "rdMB"), ("dram__bytes_write.sum", "wrMB"),
        ("lts__t_bytes.sum", "L2MB"), ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram%"),
        ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "l2%"),
        ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tc%"),
        ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", "smem%"),
        ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm%"),
        ("launch__grid_size", "grid"), ("sm__cycles_elapsed.avg.per_second", "clkGHz")]
SC = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3, "nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3,
      "hz": 1e-9, "khz": 1e-6, "mhz": 1e-3, "ghz": 1.0}
rows = list(csv.reader(open(sys.argv[1])))
hdr, units = rows[0], rows[1]
idx = {h: i for i, h in enumerate(hdr)}
names = sys.argv[2:]
tot = {}
for n, d in enumerate(rows[2:]):
    lab = names[n] if n < len(names) else d[idx["Kernel Name"]][:30]
    out = [f"{lab:10s}"]
    for m, l in WANT:
        if m not in idx:
            continue
        try:
            v = float(d[idx[m]].replace(",", "")) * SC.get(units[idx[m]].lower() if units[idx[m]] in ("hz", "Khz", "Mhz", "Ghz") else units[idx[m]], 1.0)
        except ValueError:
            continue
        tot[l] = tot.get(l, 0) + v
        out.append(f"{l}={v:.1f}" if v < 1e4 else f"{l}={v:.0f}")
    print(" ".join(out))
print("TOTAL", {k: round(v, 1) for k, v in tot.items() if k in ("us", "rdMB", "wrMB", "L2MB")})
