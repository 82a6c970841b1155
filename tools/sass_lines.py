"""Dev tool: SASS of selected source lines from `ncu --page source --csv
--print-source=cuda,sass` output: python tools/sass_lines.py src.csv FILE LINE..."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
want_file, want = sys.argv[2], set(sys.argv[3:])
hdr = cur = f = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        f = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None:
        continue
    if r[0].strip():
        cur = (f, r[0])
        continue
    if cur and cur[0] == want_file and cur[1] in want and r[7] not in ("0", "-", ""):
        print(cur[1], r[4].rjust(7), r[7].rjust(10), r[3])
