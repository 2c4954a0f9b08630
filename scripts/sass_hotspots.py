"""Join an ncu --page source --print-source sass CSV with nvdisasm -g line info.

usage: sass_hotspots.py <ncu-sass.csv> <nvdisasm -g output> <kernel-name-substring> [top]
Prints the source lines with the most warp-stall samples / executed instructions.
"""
import collections, csv, re, sys

csv_path, sass_path, kern = sys.argv[1:4]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
fn = None; cur = None; a2l = {}
for line in open(sass_path):
    m = re.match(r'\.text\.(\S+):', line.strip())
    if m:
        fn = m.group(1); continue
    m = re.search(r'//## File "([^"]+)", line (\d+)', line)
    if m:
        cur = (m.group(1).split('/')[-1], int(m.group(2))); continue
    m = re.match(r'\s*/\*([0-9a-f]{4,})\*/', line)
    if m and fn and kern in fn:
        a2l[int(m.group(1), 16)] = cur
rows = list(csv.reader(open(csv_path)))
h = rows[1]; data = rows[2:]
ai = h.index("Address"); si = h.index("Warp Stall Sampling (All Samples)")
ei = h.index("Instructions Executed"); ti = h.index("Thread Instructions Executed")
base = min(int(r[ai], 16) for r in data if r[ai].startswith("0x"))
agg = collections.defaultdict(lambda: [0.0, 0.0, 0.0]); tot = [0.0, 0.0]
stall_cols = [i for i, c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c]
stalls = collections.defaultdict(lambda: collections.Counter())
for r in data:
    if not r[ai].startswith("0x"):
        continue
    key = a2l.get(int(r[ai], 16) - base)
    s = float(r[si] or 0); e = float(r[ei] or 0); t = float(r[ti] or 0)
    agg[key][0] += s; agg[key][1] += e; agg[key][2] += t
    tot[0] += s; tot[1] += e
    for c in stall_cols:
        try:
            stalls[key][h[c]] += float(r[c] or 0)
        except ValueError:
            pass
print(f"samples {tot[0]:.0f} warp-inst {tot[1]:.3g}")
for k, v in sorted(agg.items(), key=lambda x: -x[1][0])[:top]:
    st = ", ".join(f"{n[6:]}:{c/ max(v[0],1)*100:.0f}%" for n, c in stalls[k].most_common(3))
    print(f"{str(k):32s} smp {100*v[0]/tot[0]:5.1f}% inst {100*v[1]/tot[1]:5.1f}% thr/inst {v[2]/max(v[1],1):4.1f}  [{st}]")
