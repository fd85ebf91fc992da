"""Map an ncu launch list of one eager C3 iteration (tools/one_iter.py) to layer names."""
import csv, sys
names = ["head","e0.0A","e0.0B","e0.1A","e0.1B","down0","e1.0A","e1.0B","e1.1A","e1.1B","down1","e2.0A","e2.0B","e2.1A","e2.1B","down2","e3.0A","e3.0B","e3.1A","e3.1B",
 "up2","d2.0A","d2.0B","d2.1A","d2.1B","up1","d1.0A","d1.0B","d1.1A","d1.1B","up0","d0.0A","d0.0B","d0.1A","d0.1B","tail",
 "tailT","d0.1BT","d0.1AT","d0.0BT","d0.0AT","up0T","d1.1BT","d1.1AT","d1.0BT","d1.0AT","up1T","d2.1BT","d2.1AT","d2.0BT","d2.0AT","up2T",
 "e3.1BT","e3.1AT","e3.0BT","e3.0AT","down2T","e2.1BT","e2.1AT","e2.0BT","e2.0AT","down1T","e1.1BT","e1.1AT","e1.0BT","e1.0AT","down0T","e0.1BT","e0.1AT","e0.0BT","e0.0AT","headT"]
rows = list(csv.reader(open(sys.argv[1] if len(sys.argv) > 1 else 'gpurun_out/launches_it.csv')))
hdr = None; data = []
for r in rows:
    if r and r[0] == 'ID': hdr = r; continue
    if hdr and len(r) == len(hdr): data.append(dict(zip(hdr, r)))
start = next(i for i,d in enumerate(data) if 'img2feat' in d['Kernel Name'])
tot = 0; out = []
for n, d in zip(names, data[start:start+len(names)]):
    v = float(d['Metric Value']) / 1e3; tot += v
    out.append(f"{n:7s}{v:7.1f}")
for i in range(0, len(out), 6): print("  ".join(out[i:i+6]))
print("network total us", round(tot, 1))
for d in data[start+len(names):]: print(f"  {d['Kernel Name'][:40]} {float(d['Metric Value'])/1e3:.1f}")
