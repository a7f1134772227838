"""Per-opcode and top-instruction warp-stall samples from `ncu -i REP --page source --csv --print-source sass`.
usage: ncu_source_hot.py REP [top_n]"""
import csv, collections, re, subprocess, sys
rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[1]
ia, isrc, isamp = hdr.index("Address"), hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
stall_cols = [(i, h) for i, h in enumerate(hdr) if h.startswith("stall_") or "Stall" in h and i > isamp + 1]
recs = []
for r in rows[2:]:
    if len(r) <= isamp:
        continue
    try:
        n = int(r[isamp])
    except ValueError:
        continue
    recs.append((n, r[ia], r[isrc].strip(), r))
tot = sum(n for n, *_ in recs)
byop = collections.Counter()
for n, a, s, _ in recs:
    op = re.sub(r"^@!?U?P\w+\s+", "", s).split()[0] if s else "?"
    byop[op] += n
print(f"total samples {tot}")
for op, n in byop.most_common(15):
    print(f"  {op:28s} {n:8d} {100.0 * n / tot:5.1f}%")
print("stall columns:", [h for _, h in stall_cols][:40])
names = [h for _, h in stall_cols if "Not Issued" not in h]
idx = {h: i for i, h in stall_cols}
agg = collections.defaultdict(collections.Counter)
for n, a, s, r in recs:
    op = re.sub(r"^@!?U?P\w+\s+", "", s).split()[0] if s else "?"
    for h in names:
        try:
            agg[op][h] += int(r[idx[h]] or 0)
        except ValueError:
            pass
for op, _ in byop.most_common(8):
    c = agg[op]
    print(f"{op:14s}", " ".join(f"{h[6:]}={v}" for h, v in c.most_common(6) if v))
tot_c = collections.Counter()
for op in agg:
    tot_c.update(agg[op])
print("all:", " ".join(f"{h[6:]}={v}" for h, v in tot_c.most_common(10) if v))
for op in ("SYNCS.PHASECHK.TRANS64.TRYWAIT", "BRA", "LDS.128", "STG.E.128"):
    if op in agg:
        print(f"{op:30s}", " ".join(f"{h[6:]}={v}" for h, v in agg[op].most_common(5) if v))
print("top instructions:")
for n, a, s, r in sorted(recs, key=lambda x: -x[0])[:int(sys.argv[3]) if len(sys.argv) > 3 else 0]:
    st = sorted(((int(r[idx[h]] or 0), h[6:]) for h in names if (r[idx[h]] or "0").isdigit()), reverse=True)[:3]
    print(f"  {a[-5:]} {n:5d} {s[:60]:60s} {st}")
