"""Helpers to read ncu exports here (no GPU): launch lists and --set full details."""
import csv
import subprocess
import sys
from collections import OrderedDict


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr, out = None, OrderedDict()
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            out.setdefault((int(d["ID"]), d["Kernel Name"]), {})[d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
    return out


def details(rep, filt=None):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(txt.splitlines()))
    h = r[0]
    res = []
    for row in r[1:]:
        d = dict(zip(h, row))
        res.append((d.get("Section Name", ""), d.get("Metric Name", ""), d.get("Metric Value", ""), d.get("Metric Unit", "")))
    return res


if __name__ == "__main__":
    cmd = sys.argv[1]
    if cmd == "launches":
        L = launches(sys.argv[2])
        for (i, name), m in list(L.items())[: int(sys.argv[3]) if len(sys.argv) > 3 else 40]:
            t = m.get("gpu__time_duration.sum", 0)
            rd, wr = m.get("dram__bytes_read.sum", 0), m.get("dram__bytes_write.sum", 0)
            print(f"{i:4d} {name[:60]:60s} {t/1e3:9.1f} us  rd {rd/1e9:7.3f} GB  wr {wr/1e9:7.3f} GB  {(rd+wr)/max(t,1):7.1f} GB/s")
    else:
        for sec, name, val, unit in details(sys.argv[2]):
            if name:
                print(f"{sec[:28]:28s} | {name[:50]:50s} | {val} {unit}")
