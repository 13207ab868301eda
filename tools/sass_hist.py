"""Summarise an ncu --page source --print-source sass CSV: executed warp
instructions by opcode, and the hottest basic blocks (runs of executed SASS)."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
ia, isrc, iex, ismp = h.index("Address"), h.index("Source"), h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
ops = collections.Counter(); tot = 0; stall = collections.Counter()
blocks = []; cur = None
for r in rows[2:]:
    if len(r) <= iex: continue
    try: ex = int(r[iex])
    except ValueError: continue
    src = r[isrc].strip()
    op = src.split()[0] if src else "?"
    if op.startswith("@"): op = src.split()[1]
    op = op.split(".")[0]
    ops[op] += ex; tot += ex
    stall[op] += int(r[ismp] or 0)
    if cur is None or ex != cur[0]:
        cur = [ex, 0, src, collections.Counter()]; blocks.append(cur)
    cur[1] += 1; cur[3][op] += 1
print("total warp instr", tot)
print(", ".join(f"{k} {100*v/tot:.1f}%" for k, v in ops.most_common(18)))
ts = sum(stall.values()) or 1
print("stall samples by opcode:", ", ".join(f"{k} {100*v/ts:.1f}%" for k, v in stall.most_common(10)))
blocks.sort(key=lambda b: -b[0] * b[1])
for b in blocks[:int(sys.argv[2]) if len(sys.argv) > 2 else 12]:
    print(f"== {100*b[0]*b[1]/tot:5.1f}%  exec {b[0]} x {b[1]}: {dict(b[3].most_common(7))}  | {b[2][:60]}")
