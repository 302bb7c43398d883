"""Split an ncu SASS source page (csv) into barrier-delimited regions: instructions executed,
stall samples and stall reasons per region (used to study single-CTA kernels)."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
idx = {k: i for i, k in enumerate(h)}
sc = [k for k in h if k.startswith('stall_') and 'Not Issued' not in k]
body = [r for r in rows[2:] if len(r) >= len(h)]
cuts = [i for i, r in enumerate(body) if 'BAR.SYNC' in r[1] or 'EXIT' in r[1]]
prev = 0
for c in cuts + [len(body)]:
    seg = body[prev:c + 1]
    s = sum(float(r[idx['Warp Stall Sampling (All Samples)']] or 0) for r in seg)
    ie = sum(float(r[idx['Instructions Executed']] or 0) for r in seg)
    st = {k[6:]: sum(float(r[idx[k]] or 0) for r in seg) for k in sc}
    st = {k: v for k, v in st.items() if v > 0}
    print(f"[{prev:5d},{c:5d}] instrs {len(seg):5d} executed {ie:10.0f} samples {s:5.0f} {st}")
    prev = c + 1
