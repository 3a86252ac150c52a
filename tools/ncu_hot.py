"""Print the hottest SASS instructions (warp-stall samples) of the first kernel in an
`ncu --page source --csv --print-source sass` dump, with their top stall reasons."""
import csv
import sys


def main(path, n=40):
    rows = list(csv.reader(open(path)))
    starts = [i for i, r in enumerate(rows) if r and r[0] == "Address"]
    hi = starts[0]
    end = starts[1] - 1 if len(starts) > 1 else len(rows)
    hdr, data = rows[hi], [r for r in rows[hi + 1:end] if len(r) > 5]
    ix = {h: i for i, h in enumerate(hdr)}
    key = "Warp Stall Sampling (All Samples)"
    val = lambda r: int(r[ix[key]] or 0)
    tot = sum(val(r) for r in data)
    print("total samples", tot, "instructions", len(data))
    for r in sorted(data, key=lambda r: -val(r))[:n]:
        st = {h: int(r[ix[h]]) for h in hdr if h.startswith("stall_") and "(Not" not in h and r[ix[h]] not in ("", "0")}
        top = sorted(st.items(), key=lambda x: -x[1])[:3]
        print(f"{val(r):6d} {100*val(r)/tot:5.1f}% {r[ix['Address']][-5:]} {r[ix['Source']].strip()[:58]:58s} "
              + " ".join(f"{k[6:]}={v}" for k, v in top))


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)


def opcode_mix(path):
    """Warp-level instructions executed per opcode (first kernel of the dump)."""
    rows = list(csv.reader(open(path)))
    starts = [i for i, r in enumerate(rows) if r and r[0] == "Address"]
    hi = starts[0]
    end = starts[1] - 1 if len(starts) > 1 else len(rows)
    hdr, data = rows[hi], [r for r in rows[hi + 1:end] if len(r) > 5]
    ix = {h: i for i, h in enumerate(hdr)}
    mix = {}
    for r in data:
        src = r[ix["Source"]].strip()
        toks = src.split()
        if not toks:
            continue
        op = toks[1] if toks[0].startswith("@") and len(toks) > 1 else toks[0]
        op = op.split(".")[0]
        mix[op] = mix.get(op, 0) + int(r[ix["Instructions Executed"]] or 0)
    tot = sum(mix.values())
    for op, v in sorted(mix.items(), key=lambda x: -x[1])[:25]:
        print(f"{op:12s} {v:12d} {100*v/tot:5.1f}%")
    print("total", tot)
