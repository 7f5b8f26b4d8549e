"""Join an ncu SASS source page (per-PC instructions executed) with the
cubin's line table (nvdisasm -g) to rank source lines by executed warp
instructions per search node (dev tool).

usage: sass_hotspots.py REPORT.ncu-rep LIB.so KERNEL_MANGLED NODES [TOP]
"""
import csv, io, os, re, subprocess, sys, tempfile, collections

rep, so, fn, nodes = sys.argv[1], sys.argv[2], sys.argv[3], float(sys.argv[4])
top = int(sys.argv[5]) if len(sys.argv) > 5 else 40
page = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                      capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(page)))
hi = next(i for i, r in enumerate(rows) if "Instructions Executed" in r)
hdr = rows[hi]
ia, ie, isrc = hdr.index("Address"), hdr.index("Instructions Executed"), hdr.index("Source")
pcs = []
for r in rows[hi + 1:]:
    if len(r) > ie and r[ia].startswith("0x"):
        pcs.append((int(r[ia], 16), float(r[ie] or 0), r[isrc].strip()))
base = pcs[0][0]
d = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(so)], cwd=d, capture_output=True)
cub = [f for f in os.listdir(d) if f.startswith("mcsg_kernel") and f.endswith(".cubin") and "-" not in f][0]
dis = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(d, cub)], capture_output=True, text=True).stdout
line_of = {}
cur, inside = None, False
for ln in dis.splitlines():
    if ln.startswith("//----") and ".text." in ln:
        inside = ln.split(".text.")[1].split()[0] == fn
        continue
    if not inside:
        continue
    m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
    if m:
        cur = f"{os.path.basename(m.group(1))}:{m.group(2)}"
        continue
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/", ln)
    if m:
        line_of[int(m.group(1), 16)] = cur
agg = collections.Counter()
for pc, n, _ in pcs:
    agg[line_of.get(pc - base, "?")] += n
tot = sum(agg.values())
print(f"total {tot:.4g} warp-inst, {tot / nodes:.2f} per node")
for k, v in agg.most_common(top):
    print(f"{v / nodes:7.2f}  {k}")
