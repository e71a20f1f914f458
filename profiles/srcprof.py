"""Per-source-line instruction and stall-sample shares of one kernel of an
ncu report (the --page source export with cuda,sass interleaved):
  ncu -i rep.ncu-rep --page source --csv --print-source cuda,sass --launch-skip K --launch-count 1 > x.csv
  python profiles/srcprof.py x.csv [top]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
f = None
first_fn = cur_fn = None
agg, st, src = collections.Counter(), collections.Counter(), {}
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        f = r[1].split("/")[-1]
        continue
    if r[0] == "Function Name":
        first_fn = first_fn or r[1]
        cur_fn = r[1]
        continue
    if r[0] == "Line No" or cur_fn != first_fn or r[0] == "":
        continue
    line = (f, int(r[0]))
    src[line] = r[1][:80]
    try:
        agg[line] += int(r[7])
        st[line] += int(r[4])
    except ValueError:
        pass
tot, tst = sum(agg.values()), max(1, sum(st.values()))
print(first_fn[:120])
print("total warp instructions", tot)
for k, v in sorted(agg.items(), key=lambda x: -x[1])[:top]:
    print(f"{100 * v / tot:5.1f}% inst {100 * st[k] / tst:5.1f}% stall {k[0]}:{k[1]} {src[k]}")
