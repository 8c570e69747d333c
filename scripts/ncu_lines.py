"""dev: top source lines of an ncu report (ncu -i R --page source --csv --print-source cuda,sass)."""
import csv, subprocess, sys, collections
rep = sys.argv[1]; top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
_i = lambda s: int(s) if s and s.isdigit() else 0
f = None; rows = []; hdr = None
for r in csv.reader(out.splitlines()):
    if not r: continue
    if r[0] == "File Path": f = r[1].split("/")[-1]; continue
    if r[0] == "Line No": hdr = r; continue
    if r[0] and hdr and r[0].isdigit():
        d = dict(zip(hdr[4:], r[4:]))
        rows.append((f, int(r[0]), r[1].strip()[:90], _i(d.get("# Samples")), _i(d.get("Instructions Executed"))))
ts = sum(x[3] for x in rows) or 1; ti = sum(x[4] for x in rows) or 1
print("total samples", ts, "warp instr", ti)
byfile = collections.Counter(); byfile_i = collections.Counter()
for x in rows: byfile[x[0]] += x[3]; byfile_i[x[0]] += x[4]
for k, v in byfile.most_common(): print(f"  {k}: samples {100*v/ts:.1f}% instr {100*byfile_i[k]/ti:.1f}%")
for x in sorted(rows, key=lambda x: -x[3])[:top]:
    print(f"{100*x[3]/ts:5.1f}% {100*x[4]/ti:5.1f}%  {x[0]}:{x[1]}  {x[2]}")

# per-function rollup (function = last top-level definition line above)
import re, os
CS = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2407_00023_b200", "csrc")
defs = {}
for fn in os.listdir(CS):
    starts = []
    for i, ln in enumerate(open(os.path.join(CS, fn)), 1):
        m = re.match(r"^(?:template.*)?(?:E2_\w+|__global__|static|inline|__device__)[^(]*?(\w+)\(", ln)
        if m: starts.append((i, m.group(1)))
    defs[fn] = starts
fs = collections.Counter(); fi = collections.Counter()
for f, line, _, smp, ins in rows:
    name = "?"
    for i, nm in defs.get(f, []):
        if i <= line: name = nm
    fs[f"{f}:{name}"] += smp; fi[f"{f}:{name}"] += ins
print("\nper function (samples%, instr%):")
for k, v in fs.most_common(45): print(f"  {100*v/ts:5.1f}% {100*fi[k]/ti:5.1f}%  {k}")
