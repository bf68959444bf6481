"""Per-apply DRAM bytes and durations from an in-sequence ncu capture
(--cache-control none --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum).
usage: python tools/dram_summary.py <dram.csv> [applies=4]"""
import collections, csv, re, sys


def load(path):
    rows = list(csv.reader(open(path)))
    hdr, recs = None, collections.OrderedDict()
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        key = (int(d["ID"]), re.sub(r"\(.*", "", d["Kernel Name"]).split("::")[-1][:40])
        v = float(d["Metric Value"].replace(",", ""))
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "usecond": 1,
                 "msecond": 1e3}.get(d["Metric Unit"], 1)
        recs.setdefault(key, {})[d["Metric Name"]] = v * scale
    return list(recs.items())


def applies(recs):
    """group the FMM GEMM passes into applies (7 consecutive passes after an fmm_ops launch)"""
    out, cur = [], None
    for (i, name), m in recs:
        if name.startswith("fmm_ops"):
            cur = []
            out.append(cur)
        elif name.startswith("fmm_gemm") and cur is not None:
            cur.append(m)
    return [a for a in out if a]


if __name__ == "__main__":
    recs = load(sys.argv[1])
    k = int(sys.argv[2]) if len(sys.argv) > 2 else 4
    aps = applies(recs)[-k:]
    for a in aps:
        rd = sum(m.get("dram__bytes_read.sum", 0) for m in a)
        wr = sum(m.get("dram__bytes_write.sum", 0) for m in a)
        us = sum(m.get("gpu__time_duration.sum", 0) for m in a) / 1e3
        print(f"apply: {len(a)} passes, {us:.1f} us, DRAM read {rd/1e6:.0f} MB write {wr/1e6:.0f} MB total {(rd+wr)/1e6:.0f} MB")
