"""Summarise an ncu launch-list CSV (gpu__time_duration + dram bytes) per kernel
class; writes profiles/ncu_traffic.json (DRAM bytes per launch, used by bench.py
as roofline.traffic) and prints a markdown table."""
import collections
import csv
import json
import re
import sys
from pathlib import Path

CLASS = {"k_p2g": "p2g", "k_grid_update": "grid_update", "k_g2p": "g2p", "k_adj_g2p": "g2p_adjoint",
         "k_adj_grid": "grid_adjoint", "k_eff_final": "grid_adjoint", "k_adj_p2g": "p2g_adjoint",
         "k_sort_count": "sort", "k_sort_scatter": "sort", "k_sort_blocks": "sort", "k_nb_scatter": "sort",
         "DeviceScan": "sort", "k_list_sums": "sort", "k_list_write": "sort", "k_isort_diff": "sort",
         "k_isort_arrive": "sort", "k_isort_blocks": "sort"}


def main(path, out_json):
    rows = list(csv.reader(open(path)))
    hdr = None
    recs = collections.defaultdict(lambda: collections.defaultdict(float))
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        recs[(d["ID"], d["Kernel Name"])][d["Metric Name"]] = float(d["Metric Value"].replace(",", "") or 0)
    per = collections.defaultdict(lambda: [0, 0.0, 0.0])
    kern = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for (_, name), m in recs.items():
        base = re.search(r"(k_\w+|DeviceScan\w*)", name)
        base = base.group(1) if base else name[:30]
        tm = re.search(r"k_\w+<(\(bool\))?([01])[,>]", name)  # k_x<HEAVY> / k_x<HEAVY, MINB> / k_x<(bool)H, ...>
        var = ("<H>" if tm.group(2) == "1" else "<L>") if tm else ""
        t = m.get("gpu__time_duration.sum", 0.0)
        b = m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
        k = kern[base + var]
        k[0] += 1
        k[1] += t
        k[2] += b
        cls = next((v for kk, v in CLASS.items() if base.startswith(kk)), None)
        if cls:
            c = per[cls]
            c[1] += t
            c[2] += b
    # launches per class = launches of its main kernel
    main_k = {"p2g": "k_p2g<L>", "grid_update": "k_grid_update", "g2p": "k_g2p<L>", "g2p_adjoint": "k_adj_g2p<L>",
              "grid_adjoint": "k_adj_grid", "p2g_adjoint": "k_adj_p2g<L>", "sort": "k_sort_blocks"}
    traffic = {}
    print("| kernel | launches | mean us (ncu, cold) | DRAM MB / launch | GB/s |")
    print("|---|---|---|---|---|")
    for name, (n, t, b) in sorted(kern.items(), key=lambda kv: -kv[1][1]):
        print(f"| {name} | {n} | {t / n / 1e3:.1f} | {b / n / 1e6:.2f} | {b / max(t, 1):.0f} |")
    for cls, key in main_k.items():
        n = next((v[0] for k, v in kern.items() if k.startswith(key)), 0)
        if cls == "sort":  # full and incremental sorts
            n += next((v[0] for k, v in kern.items() if k.startswith("k_isort_blocks")), 0)
        if n and cls in per:
            traffic[cls] = per[cls][2] / n
    Path(out_json).write_text(json.dumps({k: round(v) for k, v in traffic.items()}, indent=1))
    print("\ntraffic per launch (bytes):", json.dumps({k: round(v) for k, v in traffic.items()}))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
