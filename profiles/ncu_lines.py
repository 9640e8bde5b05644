"""Per-source-line stall samples / instruction counts from an ncu report
(`ncu -i REP --page source --csv -k regex:K --print-source cuda,sass`)."""
import csv, sys, collections

def main(path, top=40):
    rows = list(csv.reader(open(path)))
    f = None; hdr = None
    lines = []
    for r in rows:
        if not r: continue
        if r[0] == "File Path": f = r[1].split("/")[-1]; continue
        if r[0] == "Line No": hdr = r; continue
        if len(r) > 7 and r[0] and hdr and r[2] == "-":   # cuda line aggregate
            try:
                s = int(r[4]); n = int(r[7])
            except ValueError:
                continue
            lines.append((s, n, f, r[0], r[1][:100]))
    tot = sum(l[0] for l in lines) or 1; ti = sum(l[1] for l in lines) or 1
    print(f"total samples {tot}  instructions {ti}")
    by_file = collections.Counter()
    for l in lines: by_file[l[2]] += l[0]
    for k, v in by_file.most_common(): print(f"  {k:28s} {100*v/tot:5.1f}%")
    for s, n, fn, ln, src in sorted(lines, reverse=True)[:top]:
        print(f"{100*s/tot:5.1f}% inst {100*n/ti:5.1f}%  {fn}:{ln}  {src}")

if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
