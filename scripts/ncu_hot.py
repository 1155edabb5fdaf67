"""Summarise an ncu source-page CSV (SASS): total stall samples, the hottest instructions with
context. Usage: python scripts/ncu_hot.py gpurun_out/X_source.csv [top]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 20
hdr = rows[1]
I = {h: i for i, h in enumerate(hdr)}
data = rows[2:]
S = I["Warp Stall Sampling (All Samples)"]
tot = sum(int(r[S] or 0) for r in data)
print("total samples", tot)
for r in sorted(data, key=lambda r: -int(r[S] or 0))[:top]:
    print(r[I["Address"]][-5:], r[S].rjust(6), r[I["Instructions Executed"]].rjust(9), r[I["Source"]][:90])
