"""Top SASS lines by stall samples for one kernel of an ncu report: ncu_source.py REP KERNEL_REGEX [N]"""
import csv, subprocess, sys, io
rep, kern = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k", "regex:" + kern],
                     capture_output=True, text=True).stdout
lines = out.splitlines()
# the file is a sequence of blocks: "Kernel Name",...  then header then rows
blocks, cur = [], None
for ln in lines:
    if ln.startswith('"Kernel Name"'):
        cur = [ln]
        blocks.append(cur)
    elif cur is not None:
        cur.append(ln)
for blk in blocks[:1]:
    print(blk[0][:120])
    rows = list(csv.reader(io.StringIO("\n".join(blk[1:]))))
    hdr = rows[0]
    iS, iA, iE = hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
    data = [(int(r[iA] or 0), int(r[iE] or 0), r[0], r[iS]) for r in rows[1:] if len(r) > iA]
    tot = sum(d[0] for d in data) or 1
    print("total samples", tot)
    for s, e, a, src in sorted(data, reverse=True)[:n]:
        print(f"{100*s/tot:6.2f}% {e:>10d}  {a[-5:]}  {src.strip()}")
