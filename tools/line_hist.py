"""Dev tool: per-source-line stall samples / executed instructions from
`ncu --page source --csv --print-source=cuda,sass`."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
cur_file, cur_line, cur_src = None, None, ""
agg = collections.defaultdict(lambda: [0, 0, ""])
tot_s = tot_i = 0
hdr = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = {h: i for i, h in enumerate(r)}
        continue
    if hdr is None or len(r) < 5:
        continue
    if r[0].strip():  # a source line row
        cur_line, cur_src = r[0], r[1]
        continue
    try:
        s = int(r[4] or 0); n = int(r[7] or 0)
    except ValueError:
        continue
    k = (cur_file, cur_line)
    agg[k][0] += s; agg[k][1] += n; agg[k][2] = cur_src
    tot_s += s; tot_i += n
print("total samples", tot_s, "instr", tot_i)
for k, (s, n, src) in sorted(agg.items(), key=lambda x: -x[1][0])[: int(sys.argv[2]) if len(sys.argv) > 2 else 40]:
    print(f"{k[0]}:{k[1]:>4} samp {s/tot_s*100:5.1f}% instr {n/tot_i*100:5.1f}%  {src.strip()[:80]}")
