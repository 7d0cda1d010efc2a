"""Summarise ncu source-page SASS samples per kernel: top instructions and opcode totals."""
import csv, sys, subprocess, collections, re
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout.splitlines()
kern = None; hdr = None; data = collections.defaultdict(list)
for row in csv.reader(out):
    if not row: continue
    if row[0] == "Kernel Name": kern = row[1]; hdr = None; continue
    if row[0] == "Address": hdr = row; continue
    if hdr and kern: data[kern].append(dict(zip(hdr, row)))
for k, rows in data.items():
    tot = sum(int(r["Warp Stall Sampling (All Samples)"] or 0) for r in rows)
    print("==", k[:70], "samples", tot)
    ops = collections.Counter()
    for r in rows:
        op = r["Source"].split()[0] if r["Source"].split() else "?"
        if op.startswith("@"): op = r["Source"].split()[1]
        ops[op.split(".")[0]] += int(r["Warp Stall Sampling (All Samples)"] or 0)
    print("   by opcode:", [(o, round(v / tot, 3)) for o, v in ops.most_common(12)])
    stall_cols = [c for c in rows[0] if c.startswith("stall_")]
    sc = collections.Counter()
    for r in rows:
        for c in stall_cols:
            try: sc[c] += int(r[c] or 0)
            except: pass
    print("   stalls:", [(c, round(v / tot, 3)) for c, v in sc.most_common(8)])
    top = sorted(range(len(rows)), key=lambda i: -int(rows[i]["Warp Stall Sampling (All Samples)"] or 0))[:int(sys.argv[2]) if len(sys.argv) > 2 else 25]
    for i in sorted(top):
        r = rows[i]
        st = sorted(((int(r[c] or 0), c) for c in stall_cols), reverse=True)[:2]
        print("   %5d %6.3f  %-60s %s" % (i, int(r["Warp Stall Sampling (All Samples)"] or 0) / tot, r["Source"].strip()[:60], [(c[6:], v) for v, c in st if v]))
