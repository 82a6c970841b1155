"""Dev tool: aggregate an ncu --page source --print-source=sass CSV by opcode."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
by_op = collections.defaultdict(lambda: [0, 0, 0])
tot_s = tot_i = 0
body = rows[2:]
for r in body:
    if len(r) < len(hdr) - 1:
        continue
    src = r[ix["Source"]].strip()
    op = src.split()[0] if src else "?"
    if op.startswith("@"):
        op = src.split()[1]
    op = op.split(".")[0]
    s = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    n = int(r[ix["Instructions Executed"]] or 0)
    th = int(r[ix["Thread Instructions Executed"]] or 0)
    by_op[op][0] += s; by_op[op][1] += n; by_op[op][2] += th
    tot_s += s; tot_i += n
print(f"total samples {tot_s} warp-instr {tot_i}")
for op, (s, n, th) in sorted(by_op.items(), key=lambda x: -x[1][1])[:40]:
    print(f"{op:12s} instr {n/tot_i*100:5.1f}%  stall-samples {s/tot_s*100:5.1f}%  avg-threads {th/max(n,1):5.1f}")
if len(sys.argv) > 2:
    # hottest individual instructions
    hot = sorted(body, key=lambda r: -int(r[ix["Warp Stall Sampling (All Samples)"]] or 0) if len(r) >= len(hdr)-1 else 0)[:int(sys.argv[2])]
    for r in hot:
        print(r[ix["Address"]][-5:], r[ix["Warp Stall Sampling (All Samples)"]], r[ix["Instructions Executed"]], r[ix["Source"]].strip()[:70])
