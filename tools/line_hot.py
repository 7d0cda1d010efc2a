"""Per-source-line warp-stall samples from an ncu report (cuda,sass view).
usage: line_hot.py report.ncu-rep [kernel-substring] [top] [source-file-for-text]"""
import csv, subprocess, sys, collections
rep = sys.argv[1]
ksub = sys.argv[2] if len(sys.argv) > 2 else ""
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
src = open(sys.argv[4]).read().split("\n") if len(sys.argv) > 4 else None
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout.splitlines()
texts = {}; func = None; hdr = None; per = collections.defaultdict(collections.Counter); stall = collections.defaultdict(dict)
for row in csv.reader(out):
    if not row: continue
    if row[0] == "Function Name": func = row[1]; continue
    if row[0] == "Line No": hdr = row; continue
    if hdr is None or func is None or ksub not in func: continue
    if row[0] and row[0].isdigit():
        ln = int(row[0]); v = int(row[4]) if row[4].isdigit() else 0
        per[func][ln] += v
        texts[ln] = row[1]
        cols = {hdr[i]: row[i] for i in range(len(hdr)) if hdr[i].startswith("stall_") and "Not Issued" not in hdr[i]}
        stall[func][ln] = sorted(((int(x) if x.isdigit() else 0, k[6:]) for k, x in cols.items()), reverse=True)[:3]
for f, c in per.items():
    tot = sum(c.values())
    print("==", f[:90], "samples", tot)
    for ln, v in c.most_common(top):
        text = texts.get(ln, "").strip()[:70]
        print("  %5d %6.3f  %-70s %s" % (ln, v / tot, text, [(k, n) for n, k in stall[f][ln] if n]))
