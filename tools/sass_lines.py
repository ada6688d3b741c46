"""Attribute ncu per-instruction stall samples (source page, SASS view) to CUDA source lines using
nvdisasm line info of the same cubin. Usage: sass_lines.py REPORT.ncu-rep KERNEL.cubin FUNC [top]"""
import csv, io, re, subprocess, sys, collections
rep, cubin, func = sys.argv[1:4]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
full = subprocess.run(["nvdisasm", "-gi", cubin], capture_output=True, text=True).stdout
sec = re.search(r"\.section\s+\.text\." + re.escape(func) + r".*?(?=\n\s*\.section|\Z)", full, re.S)
dis = sec.group(0) if sec else ""
line_of = {}
inner = outer = "?"
new_group = True
for ln in dis.splitlines():
    m = re.search(r'//## File "([^"]+)", line (\d+)(?: inlined at "([^"]+)", line (\d+))?', ln)
    if m:
        loc = f"{m.group(1).split('/')[-1]}:{m.group(2)}"
        if new_group:  # the first marker of a group is the innermost location, the last the kernel's
            inner = loc
            new_group = False
        outer = loc
        continue
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", ln)
    if m:
        line_of[int(m.group(1), 16)] = (inner, outer, m.group(2).strip())
        new_group = True
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
ai, si = h.index("Address"), h.index("Warp Stall Sampling (All Samples)")
base = int(rows[2][ai], 16)
agg_in, agg_out = collections.Counter(), collections.Counter()
stall_cols = [i for i, c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c]
why = collections.defaultdict(collections.Counter)
tot = 0
for r in rows[2:]:
    if len(r) <= si or not r[ai].startswith("0x"):
        break  # (next kernel's block)
    off = int(r[ai], 16) - base
    s = int(r[si] or 0)
    tot += s
    inn, outr, ins = line_of.get(off, ("?", "?", ""))
    agg_in[inn] += s
    agg_out[outr] += s
    for i in stall_cols:
        v = int(r[i] or 0)
        if v:
            why[inn][h[i]] += v
print("total samples", tot)
print("-- by innermost line")
for k, v in agg_in.most_common(top):
    print(f"{v:6d} {k:28s} {dict(why[k].most_common(3))}")
print("-- by kernel-level line")
for k, v in agg_out.most_common(top // 2):
    print(f"{v:6d} {k}")
