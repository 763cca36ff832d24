"""Per-kernel summary of an ncu --metrics launch list (csv): launches, mean
time, DRAM read/write per launch. Usage: summarize_launches.py file.csv"""
import csv
import io
import sys
from collections import defaultdict

UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "us": 1, "usecond": 1, "nsecond": 1e-3,
        "msecond": 1e3, "ms": 1e3, "%": 1, "sector": 1, "": 1}


def load(path):
    txt = open(path).read()
    rows = list(csv.DictReader(io.StringIO(txt[txt.index('"ID"'):])))
    per = defaultdict(lambda: defaultdict(dict))
    for r in rows:
        v = float(r["Metric Value"].replace(",", "")) * UNIT.get(r["Metric Unit"], 1)
        per[r["ID"]][r["Metric Name"]] = v
        per[r["ID"]]["name"] = r["Kernel Name"]
    return per


def summarize(path):
    per = load(path)
    agg = defaultdict(list)
    for lid, m in per.items():
        agg[m["name"].split("(")[0]].append(m)
    out = {}
    for name, ms in agg.items():
        def avg(k):
            vals = [m[k] for m in ms if k in m]
            return sum(vals) / len(vals) if vals else None
        out[name] = dict(launches=len(ms), us=avg("gpu__time_duration.sum"), dram_read=avg("dram__bytes_read.sum"),
                         dram_write=avg("dram__bytes_write.sum"), l2_sectors=avg("lts__t_sectors.sum"),
                         l1_hit=avg("l1tex__t_sector_hit_rate.pct"))
    return out


if __name__ == "__main__":
    for name, s in summarize(sys.argv[1]).items():
        t = s["us"]
        dr = (s["dram_read"] or 0) + (s["dram_write"] or 0)
        print(f"{s['launches']:4d} x {t:9.2f} us  DRAM {dr / 1e6:9.2f} MB  ({dr / 1e3 / t:7.1f} GB/s)  {name[-60:]}")
