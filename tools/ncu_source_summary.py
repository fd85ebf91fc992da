"""Summarise an `ncu --page source --csv --print-source sass` export: per kernel, the SASS
instructions with the most excessive shared-memory wavefronts and the most stall samples.
usage: python tools/ncu_source_summary.py SRC.csv [top]"""
import csv, sys
top = int(sys.argv[2]) if len(sys.argv) > 2 else 8
rows = list(csv.reader(open(sys.argv[1])))
blocks, cur = [], None
for r in rows:
    if r and r[0] == "Kernel Name":
        cur = {"name": r[1][:70], "rows": [], "hdr": None}; blocks.append(cur); continue
    if cur is None or not r: continue
    if r[0] == "Address": cur["hdr"] = r; continue
    if cur["hdr"]: cur["rows"].append(dict(zip(cur["hdr"], r)))
def f(d, k):
    try: return float(d.get(k, "0").replace(",", "") or 0)
    except ValueError: return 0.0
for b in blocks:
    rs = b["rows"]
    exc = sum(f(d, "L1 Wavefronts Shared Excessive") for d in rs)
    smp = sum(f(d, "Warp Stall Sampling (All Samples)") for d in rs)
    ins = sum(f(d, "Instructions Executed") for d in rs)
    print(f"== {b['name']}  instr={ins:.3g} stall_samples={smp:.0f} shared_excessive_wavefronts={exc:.3g}")
    for d in sorted(rs, key=lambda d: -f(d, "L1 Wavefronts Shared Excessive"))[:top]:
        if f(d, "L1 Wavefronts Shared Excessive") <= 0: break
        print(f"   excess {f(d,'L1 Wavefronts Shared Excessive'):10.0f} ideal {f(d,'L1 Wavefronts Shared Ideal'):10.0f} {d['Address']} {d['Source'][:70]}")
    for d in sorted(rs, key=lambda d: -f(d, "Warp Stall Sampling (All Samples)"))[:top]:
        print(f"   stall {f(d,'Warp Stall Sampling (All Samples)'):7.0f} ({100*f(d,'Warp Stall Sampling (All Samples)')/max(smp,1):4.1f}%) exec {f(d,'Instructions Executed'):9.0f} {d['Address']} {d['Source'][:70]}")
