"""Top SASS instructions by warp-stall samples from
`ncu -i REP --page source --csv -k regex:K --print-source sass` (run here, no GPU).
Also sums samples per opcode class and per coarse program region (split at BAR/barrier.cluster)."""
import csv, sys, collections

def main(path, top=40):
    rows = list(csv.reader(open(path, errors="replace")))
    hdr = rows[1]
    iS, iN, iE = hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
    ins = []
    for r in rows[2:]:
        if len(r) <= iE: continue
        try: ins.append((r[0], r[iS].strip(), int(r[iN] or 0), int(r[iE] or 0)))
        except ValueError: pass
    tot = sum(x[2] for x in ins) or 1
    print(f"total samples {tot}, instructions {len(ins)}")
    byop = collections.Counter()
    for a, s, n, e in ins: byop[s.split()[0] if not s.startswith("@") else s.split()[1]] += n
    print("by opcode:", ", ".join(f"{k} {100*v/tot:.1f}%" for k, v in byop.most_common(14)))
    reg = 0; regs = collections.Counter(); rstart = {0: 0}
    for k, (a, s, n, e) in enumerate(ins):
        if "BAR" in s or "UCGABAR" in s or "barrier" in s.lower():
            reg += 1; rstart[reg] = k
        regs[reg] += n
    print("by region (split at barriers):", ", ".join(f"r{k}@{rstart[k]} {100*v/tot:.1f}%" for k, v in sorted(regs.items())))
    for k in sorted(range(len(ins)), key=lambda k: -ins[k][2])[:top]:
        a, s, n, e = ins[k]
        print(f"{100*n/tot:5.1f}%  #{k:5d} exec {e:9d}  {s[:90]}")

if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
