"""Top stall lines of a `tools/ncu_source.sh` export with a few lines of context:
python tools/ncu_top_stalls.py gpurun_out/<name>.sass.csv [n_top] [context]"""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
ntop = int(sys.argv[2]) if len(sys.argv) > 2 else 12
ctx = int(sys.argv[3]) if len(sys.argv) > 3 else 6
hdr, data = rows[1], rows[2:]
ia, isamp = hdr.index('Source'), hdr.index('Warp Stall Sampling (All Samples)')
val = lambda r: int(r[isamp]) if len(r) > isamp and r[isamp].isdigit() else 0
tot = sum(val(r) for r in data)
print(rows[0][1][:120], '\ntotal samples', tot, 'instructions', len(data))
top = sorted(range(len(data)), key=lambda i: -val(data[i]))[:ntop]
for c in top:
    print(f'---- line {c}: {val(data[c])} samples ({100 * val(data[c]) / tot:.1f}%)')
    for i in range(max(0, c - ctx), min(len(data), c + 2)):
        print(f'{i:6d} {val(data[i]):6d}  {data[i][ia].strip()[:110]}')
