"""Per-source-line shared-memory wavefronts (ideal vs actual) from an ncu report."""
import csv, subprocess, sys, collections
rep, ksub = sys.argv[1], sys.argv[2]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout.splitlines()
func = None; hdr = None; rows = []
for row in csv.reader(out):
    if not row: continue
    if row[0] == "Function Name": func = row[1]; continue
    if row[0] == "Line No": hdr = row; continue
    if hdr and func and ksub in func and row[0].isdigit():
        d = dict(zip(hdr, row))
        def num(k):
            v = d.get(k, "0").replace(",", "")
            try: return float(v)
            except: return 0.0
        rows.append((num("L1 Wavefronts Shared"), num("L1 Wavefronts Shared Ideal"), int(row[0]), row[1].strip()[:80]))
tot = sum(r[0] for r in rows)
print("total shared wavefronts", tot)
for w, ideal, ln, txt in sorted(rows, reverse=True)[:15]:
    print("%5d %7.3f ideal %7.3f  %s" % (ln, w / tot, ideal / tot, txt))
