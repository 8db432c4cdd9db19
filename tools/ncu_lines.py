# aggregate an ncu "--page source --print-source cuda,sass --csv" dump per CUDA source line -- dev helper
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
fname, hdr, out = None, None, []
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 5 or r[2] != "-":
        continue
    d = dict(zip(hdr[2:], r[2:]))
    def g(k):
        try:
            return int(d.get(k, "0") or 0)
        except ValueError:
            return 0
    allv = g("Warp Stall Sampling (All Samples)")
    bar = g("stall_barrier")
    out.append((allv - bar, allv, fname, r[0], r[1].strip()[:90],
                {k: g(k) for k in hdr if k.startswith("stall_") and "Not Issued" not in k and k != "stall_barrier"}))
tot = sum(o[0] for o in out)
print("non-barrier samples", tot)
for o in sorted(out, key=lambda x: -x[0])[:top]:
    st = sorted(o[5].items(), key=lambda x: -x[1])[:3]
    print(f"{o[0]:7d} {100*o[0]/max(tot,1):5.1f}% {o[2]}:{o[3]:>5} {o[4]:90s} " + " ".join(f"{k[6:]}={v}" for k, v in st))
