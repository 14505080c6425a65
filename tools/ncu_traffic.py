"""Extract per-launch DRAM traffic from an ncu --set full report into
profiles/ncu_traffic.json (bytes per element, so bench.py can scale it)."""
import csv, io, json, subprocess, sys
n = int(sys.argv[1])
rows, hdr, units = [], None, None
for rep in sys.argv[2:]:
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(io.StringIO(raw)))
    hdr, units = rr[0], rr[1]
    rows += [r + [rep] for r in rr[2:]]
rows = [hdr, units] + rows
def val(r, k):
    v = float(r[hdr.index(k)]); u = units[hdr.index(k)]
    return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
acc = {}
for r in rows[2:]:
    name = r[hdr.index("Kernel Name")]
    b = val(r, "dram__bytes_read.sum") + val(r, "dram__bytes_write.sum")
    t = float(r[hdr.index("gpu__time_duration.sum")])
    key = ("round_log" if any(k in name for k in ("rl_fused", "rl_stream", "rl_expand", "rl_scan"))
           else "replay" if any(k in name for k in ("rp_fused", "rp_stream", "rp_tile")) else name)
    acc.setdefault(key, {}).setdefault(name.split("(")[0], []).append((b, t, r[-1]))
out = {}
for key, kern in acc.items():
    per = {k: sum(b for b, _, _ in v) / len(v) for k, v in kern.items()}
    out[key] = {"dram_bytes_per_elem": sum(per.values()) / n, "n_profiled": n, "per_kernel_bytes": per,
                "per_kernel_us": {k: sum(t for _, t, _ in v) / len(v) for k, v in kern.items()},
                "reports": sorted({rp for v in kern.values() for _, _, rp in v})}
print(json.dumps(out, indent=1))
