"""Per-region stall breakdown from an ncu source page CSV (development aid).
usage: ncu_regions.py src.csv start:end[:name] ..."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr, data = rows[1], rows[2:]
ia, iex, iss = hdr.index("Address"), hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
base = int(data[0][ia], 16)
tot = sum(float(r[iss] or 0) for r in data)
for spec in sys.argv[2:]:
    p = spec.split(":")
    lo, hi = int(p[0], 16), int(p[1], 16)
    sel = [r for r in data if lo <= int(r[ia], 16) - base < hi]
    ss = sum(float(r[iss] or 0) for r in sel)
    ex = sum(float(r[iex] or 0) for r in sel)
    br = {h: sum(float(r[hdr.index(h)] or 0) for r in sel) for h in stalls}
    top = sorted(br.items(), key=lambda t: -t[1])[:6]
    print(f"{p[2] if len(p) > 2 else spec}: samples {ss:.0f} ({ss / tot * 100:.1f}%) inst {ex:.0f} | " +
          " ".join(f"{h[6:]}={v / max(ss, 1) * 100:.0f}%" for h, v in top))
