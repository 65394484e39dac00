"""Aggregate an ncu 'cuda,sass' source CSV to per-CUDA-line instruction and
stall shares (dev tool for reading profiles/)."""
import csv
import sys


def main(path, top=40):
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
    hdr = rows[h]
    ie = hdr.index("Instructions Executed")
    ss = hdr.index("Warp Stall Sampling (All Samples)")
    cols = {n: i for i, n in enumerate(hdr) if n.startswith("stall_") and "Not Issued" not in n}
    lines = []
    cur = None
    for r in rows[h + 1:]:
        if not r:
            continue
        if r[0] and len(r) == len(hdr):   # a CUDA line with aggregated metrics
            try:
                st = {n: int(r[i] or 0) for n, i in cols.items()}
                lines.append((int(r[ie] or 0), int(r[ss] or 0), r[0], r[1][:100], st))
            except ValueError:
                pass
    tot = sum(x[0] for x in lines) or 1
    tots = sum(x[1] for x in lines) or 1
    print(f"total warp-inst {tot:.3e}  stall samples {tots}")
    for x in sorted(lines, key=lambda x: -x[1])[:top]:
        topst = sorted(x[4].items(), key=lambda kv: -kv[1])[:3]
        ts = " ".join(f"{k[6:]}={v/max(x[1],1)*100:.0f}%" for k, v in topst if v)
        print(f"{x[0]/tot*100:5.1f}%inst {x[1]/tots*100:5.1f}%smp L{x[2]:>4} {x[3]:<70} {ts}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
