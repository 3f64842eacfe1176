"""Aggregates an ncu SASS source-page CSV (warp-stall samples per instruction)
by CUDA source line, using nvdisasm --print-line-info of the kernel's cubin.
  python tools/ncu_lines.py src.csv lines.txt kernel_mangled [top]"""
import csv, re, sys, collections
src_csv, lines_txt, kern = sys.argv[1:4]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
# offset -> (file, line)
omap = {}
cur = None
inside = False
for ln in open(lines_txt):
    if ln.startswith(".text." + kern + ":"):
        inside = True
        continue
    if inside and ln.startswith(".") and not ln.startswith(".L"):
        if not ln.startswith(".text." + kern):
            break
    if not inside:
        continue
    m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
    if m:
        cur = (m.group(1).split("/")[-1], int(m.group(2)))
        continue
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/", ln)
    if m and cur:
        omap[int(m.group(1), 16)] = cur
rows = list(csv.reader(open(src_csv)))
hdr = rows[1]
ia, ist, ie = hdr.index("Address"), hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
recs = []
for r in rows[2:]:
    try:
        recs.append((int(r[ia], 16), int(r[ist] or 0), int(r[ie] or 0)))
    except Exception:
        pass
base = min(a for a, _, _ in recs)
agg = collections.Counter()
ex = collections.Counter()
for a, s, e in recs:
    key = omap.get(a - base, ("?", 0))
    agg[key] += s
    ex[key] += e
tot = sum(agg.values())
print(f"total samples {tot}")
for (f, l), s in agg.most_common(top):
    print(f"{f}:{l}  {s}  {100*s/tot:.1f}%  inst {ex[(f, l)]}")

# stall-reason totals, and per-line breakdown for the top lines
if len(sys.argv) > 5:
    cols = [i for i, c in enumerate(hdr) if c.startswith("stall_") and "Not Issued" not in c]
    tot_r = collections.Counter()
    per_line = collections.defaultdict(collections.Counter)
    for r in rows[2:]:
        try:
            a = int(r[ia], 16)
        except Exception:
            continue
        key = omap.get(a - base, ("?", 0))
        for i in cols:
            v = int(r[i] or 0)
            tot_r[hdr[i]] += v
            per_line[key][hdr[i]] += v
    print("stall totals:", ", ".join(f"{k[6:]} {v}" for k, v in tot_r.most_common(10)))
    for (f, l), s in agg.most_common(int(sys.argv[5])):
        print(f"{f}:{l}", ", ".join(f"{k[6:]} {v}" for k, v in per_line[(f, l)].most_common(4)))
