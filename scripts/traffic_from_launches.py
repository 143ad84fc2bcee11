"""ncu launch list of the bench command -> per-kernel shares of one fwd+inv
step and the ALT stages' DRAM traffic per direction (what bench.py reports
as roofline.traffic).

  python scripts/traffic_from_launches.py profiles/r02_launches_bench_n1024.csv \
      > profiles/r02_traffic_n1024.json

The list comes from
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
      --clock-control none --csv python bench.py --steps 2 --warmup 1 ...
The first forward direction is the first run of consecutive ALT launches
(alt_chain_kernel / alt_stage_kernel) after a coef_pack launch, the first
inverse the first run that ends in a coef_unpack launch."""
import csv
import json
import re
import sys

path = sys.argv[1]
rows = {}
order = []
with open(path) as fh:
    lines = [l for l in fh if l.startswith('"')]
for r in csv.DictReader(lines):
    i = int(r["ID"])
    if i not in rows:
        rows[i] = {"name": r["Kernel Name"]}
        order.append(i)
    rows[i][r["Metric Name"]] = float(r["Metric Value"].replace(",", "")) * \
        ({"ns": 1e-3, "us": 1.0, "ms": 1e3, "s": 1e6}.get(r["Metric Unit"], 1.0)
         if r["Metric Name"].startswith("gpu__time") else
         {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(r["Metric Unit"], 1.0))


def short(name):
    for k in ("alt_chain_kernel", "alt_stage_kernel", "sht_synth", "sht_anal", "coef_pack",
              "coef_unpack"):
        if k in name:
            return k
    return "other"


seq = [(i, short(rows[i]["name"])) for i in order]


def alt_run(start_kind, end_kind):
    """first maximal run of ALT launches preceded by start_kind / followed by end_kind"""
    k = 0
    while k < len(seq):
        if seq[k][1].startswith("alt_"):
            j = k
            while j < len(seq) and seq[j][1].startswith("alt_"):
                j += 1
            before = seq[k - 1][1] if k else ""
            after = seq[j][1] if j < len(seq) else ""
            if (start_kind is None or before == start_kind) and (end_kind is None or after == end_kind):
                return [s[0] for s in seq[k:j]]
            k = j
        else:
            k += 1
    return []


def summarize(ids):
    t = sum(rows[i]["gpu__time_duration.sum"] for i in ids)
    rd = sum(rows[i]["dram__bytes_read.sum"] for i in ids)
    wr = sum(rows[i]["dram__bytes_write.sum"] for i in ids)
    return {"launches": len(ids), "ids": [ids[0], ids[-1]] if ids else [],
            "chain_kernel_launches": sum("alt_chain" in rows[i]["name"] for i in ids),
            "time_us": t, "dram_read_bytes": rd, "dram_write_bytes": wr,
            "traffic_bytes": rd + wr}


fwd = alt_run("coef_pack", None)
inv = alt_run(None, "coef_unpack")
m = re.search(r"_n(\d+)", path)
out = {"n": int(m.group(1)) if m else None,
       "source": f"{path} (ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,"
                 "dram__bytes_write.sum --clock-control none; scripts/traffic_from_launches.py)",
       "fwd": summarize(fwd), "inv": summarize(inv)}
out["traffic_bytes_per_direction"] = (out["fwd"]["traffic_bytes"] + out["inv"]["traffic_bytes"]) / 2
# one fwd+inv step: from the forward's coef_pack to the inverse's coef_unpack
if fwd and inv:
    lo = order.index(fwd[0]) - 1
    hi = order.index(inv[-1]) + 1
    # the step whose inverse follows this forward: take forward + following launches up to
    # the first coef_unpack after it
    k = order.index(fwd[-1])
    while k < len(order) and short(rows[order[k]]["name"]) != "coef_unpack":
        k += 1
    step = order[lo:k + 1]
    tot = sum(rows[i]["gpu__time_duration.sum"] for i in step)
    share = {}
    for i in step:
        share[short(rows[i]["name"])] = share.get(short(rows[i]["name"]), 0.0) + \
            rows[i]["gpu__time_duration.sum"]
    out["step"] = {"launches": len(step), "time_us": tot,
                   "share_us": {k2: round(v, 1) for k2, v in sorted(share.items())},
                   "share_pct": {k2: round(100 * v / tot, 1) for k2, v in sorted(share.items())}}
print(json.dumps(out, indent=1))
