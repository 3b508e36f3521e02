"""Summarise an ncu source page (SASS): samples / instructions per opcode,
stall reasons, and the hottest lines.  usage: sass_hot.py report.ncu-rep [nlines]"""
import collections, csv, io, re, subprocess, sys
rep = sys.argv[1]; nl = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]; data = []
for r in rows[2:]:  # first kernel only
    if r and r[0] == "Kernel Name":
        break
    if len(r) == len(hdr):
        data.append(r)
iS = hdr.index("Warp Stall Sampling (All Samples)"); iE = hdr.index("Instructions Executed")
stall_cols = [i for i, h in enumerate(hdr) if h.startswith('stall_') and 'Not Issued' not in h]
num = lambda x: int(x) if x.isdigit() else 0
cat = collections.Counter(); inst = collections.Counter(); st = collections.Counter()
for r in data:
    op = re.sub(r'^@!?U?P\w+\s+', '', r[1].strip())
    base = op.split()[0].split('.')[0] if op else ''
    cat[base] += num(r[iS]); inst[base] += num(r[iE])
    for i in stall_cols: st[hdr[i]] += num(r[i])
tot = sum(cat.values()); ti = sum(inst.values())
print("warp instructions", ti, "samples", tot)
for k, v in cat.most_common(14): print(f"  {k:10s} {100*v/tot:5.1f}% samples {100*inst[k]/ti:5.1f}% inst")
ts = sum(st.values())
print("stalls:", ", ".join(f"{k[6:]} {100*v/ts:.1f}%" for k, v in st.most_common(8)))
for r in sorted(data, key=lambda r: -num(r[iS]))[:nl]:
    top = sorted(((num(r[i]), hdr[i][6:]) for i in stall_cols if num(r[i])), reverse=True)[:2]
    print(f"  {r[0][-5:]} {r[1].strip()[:64]:64s} {r[iS]:>6s} {r[iE]:>10s} {top}")
