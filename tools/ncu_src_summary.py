"""Summarise an ncu --page source --csv dump: instruction mix, stall reasons, hot blocks."""
import collections
import csv
import sys


def main(path, top=25):
    rows = list(csv.reader(open(path)))
    hdr = rows[1]
    data = [r for r in rows[2:] if len(r) >= len(hdr)]
    iS, iE = hdr.index("Source"), hdr.index("Instructions Executed")
    iW = hdr.index("Warp Stall Sampling (All Samples)")
    stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
    tot, samp, st = collections.Counter(), collections.Counter(), collections.Counter()
    for r in data:
        src = r[iS].strip().split()
        op = (src[1] if src and src[0].startswith("@") else (src[0] if src else "?")).split(".")[0]
        e, s = int(r[iE] or 0), int(r[iW] or 0)
        tot[op] += e
        samp[op] += s
        for i in stall_cols:
            st[hdr[i]] += int(r[i] or 0)
    te, ts = sum(tot.values()), sum(samp.values())
    print(f"warp instructions {te}  stall samples {ts}")
    for op, c in tot.most_common(top):
        print(f"  {op:10s} {c:10d} {c / te:.3f}  samples {samp[op] / ts:.3f}")
    print("stalls:", ", ".join(f"{k[6:]} {v / ts:.2f}" for k, v in st.most_common(10)))
    blocks, cur = [], None
    for r in data:
        e, s = int(r[iE] or 0), int(r[iW] or 0)
        if cur and cur[1] == e:
            cur[2] += 1
            cur[3] += s
            cur[5] = r[iS].strip()[:40]
        else:
            cur = [r[0][-5:], e, 1, s, r[iS].strip()[:40], r[iS].strip()[:40]]
            blocks.append(cur)
    print("blocks (>0.5% of instructions): addr exec n inst% samp%")
    for b in blocks:
        if b[1] * b[2] > 0.005 * te:
            print(f"  {b[0]} {b[1]:8d} {b[2]:4d} {100 * b[1] * b[2] / te:5.1f} {100 * b[3] / ts:5.1f}  {b[4]} | {b[5]}")


if __name__ == "__main__":
    main(sys.argv[1])
