"""Dev tool: length of the trace kernel's inner step loop in a cuobjdump -sass listing.
The loop is closed by the VOTE.ANY + backwards BRA of the inner step loop."""
import re, sys
lines = [l for l in open(sys.argv[1]) if re.search(r'/\*[0-9a-f]{4}\*/', l)]
ins = []
for l in lines:
    m = re.search(r'/\*([0-9a-f]{4,})\*/\s+(.*?);', l)
    if m:
        ins.append((int(m.group(1), 16), m.group(2).strip()))
addr = {a: i for i, (a, _) in enumerate(ins)}
best = None
for i, (a, t) in enumerate(ins):
    m = re.search(r'BRA\s+(?:`\(\.L_x_\d+\)|0x([0-9a-f]+))', t)
    if 'VOTE.ANY' in ins[i - 2][1] or 'VOTE.ANY' in ins[i - 3][1]:
        m2 = re.search(r'0x([0-9a-f]+)', t)
        if m2 and int(m2.group(1), 16) < a:
            tgt = addr.get(int(m2.group(1), 16))
            if tgt is not None:
                print(f"back-edge at {a:#x} -> {int(m2.group(1),16):#x}: {i - tgt + 1} instructions (incl. skipped blocks)")
