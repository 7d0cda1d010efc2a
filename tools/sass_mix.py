"""Per-kernel SASS instruction mix of libedaa_cuda.so (cuobjdump -sass): which engines the
kernels use (DMMA = fp64 tensor pipe, UTMALDG = TMA loads, SYNCS = mbarrier, UTC*MMA/LDTM =
tcgen05/TMEM).  Usage: python tools/sass_mix.py [lib.so] > profiles/roundN/sass_mix.md"""
import collections
import re
import subprocess
import sys

lib = sys.argv[1] if len(sys.argv) > 1 else "paper_2209_11002_b200/libedaa_cuda.so"
out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
KEYS = ["DMMA", "DFMA", "DADD", "DMUL", "F2F", "UTMALDG", "SYNCS", "BAR", "LDS", "STS", "LDGSTS", "LDG", "STG",
        "RED", "ATOM", "SHFL", "MUFU", "UTCIMMA", "UTCHMMA", "UTCQMMA", "LDTM", "USETMAXREG"]
per = collections.OrderedDict()
cur = None
for line in out.splitlines():
    m = re.match(r"\s*Function : (\S+)", line)
    if m:
        cur = m.group(1)
        per[cur] = collections.Counter()
        continue
    m = re.match(r"\s+/\*[0-9a-f]+\*/\s+(?:@!?U?P\d+\s+)?([A-Z0-9_]+)", line)
    if m and cur:
        op = m.group(1)
        per[cur]["total"] += 1
        for k in KEYS:
            if op.startswith(k):
                per[cur][k] += 1
                break


def demangle(names):
    r = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True).stdout.splitlines()
    return dict(zip(names, r))


dm = demangle(list(per))
groups = collections.OrderedDict()
for name, c in per.items():
    d = dm.get(name, name)
    d = re.sub(r"\(edaa::PassArgs.*", "", d).replace("void edaa::", "").replace("pass_impl::", "").replace("(anonymous namespace)::", "")
    key = re.sub(r"\(.*", "", re.sub(r"<.*", "", d)).replace("void ", "").replace("edaa::", "")
    if "k_pass_b64" in d:
        key = "k_pass_b64 (B pass, 64-pixel logical tiles)"
    elif "k_pass" in d:
        m = re.search(r"k_pass<(?:\(int\))?(\d), (?:\(int\))?(\d+), (?:\(int\))?(\d), (\w+), ", d)
        mode = {"0": "init", "1": "A", "2": "B", "3": "obj"}[m.group(1)] if m else "?"
        key = "k_pass<%s, %s>" % (mode, m.group(4) if m else "?")
    g = groups.setdefault(key, [0, collections.Counter()])
    g[0] += 1
    g[1].update(c)
tot = collections.Counter()
print("# SASS instruction mix of %s\n" % lib.split("/")[-1])
print("Counts are static instructions summed over a kernel's instantiations (`cuobjdump -sass`, sm_100a).\n")
cols = [k for k in KEYS if any(g[1][k] for g in groups.values())]
print("| kernel | variants | instructions | " + " | ".join(cols) + " |")
print("|---|---|---|" + "---|" * len(cols))
for k, (n, c) in groups.items():
    tot.update(c)
    print("| `%s` | %d | %d | " % (k, n, c["total"]) + " | ".join(str(c[x]) if c[x] else "" for x in cols) + " |")
print("| **all** | %d | %d | " % (sum(g[0] for g in groups.values()), tot["total"]) + " | ".join(str(tot[x]) for x in cols) + " |")
print("\ntcgen05 / TMEM mnemonics (UTC*MMA, LDTM): %d — the contractions are fp64 (DMMA.884); tcgen05 has no fp64 kind."
      % (tot["UTCIMMA"] + tot["UTCHMMA"] + tot["UTCQMMA"] + tot["LDTM"]))
