"""Summarise an ncu report (raw page) and a launch-list CSV into JSON for
profiles/ (the evidence bench.py's roofline.traffic reads)."""
import csv, io, json, subprocess, sys

WANT = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "lts__t_bytes.sum": "l2_bytes",
    "launch__registers_per_thread": "registers",
    "launch__occupancy_limit_registers": "occ_limit_regs",
    "launch__occupancy_limit_shared_mem": "occ_limit_smem",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active_pct",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "sm__inst_executed.sum": "inst_executed",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active": "fp64_pipe_pct",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_throughput_pct",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
}


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units, v = rows[0], rows[1], rows[2]
    d = {}
    for i, name in enumerate(h):
        if name in WANT:
            d[WANT[name]] = {"value": v[i], "unit": units[i]}
        if "warps_issue_stalled" in name and name.endswith("_per_issue_active.ratio"):
            d.setdefault("stalls_per_issue", {})[name.split("stalled_")[1].split("_per")[0]] = float(v[i])
    return d


def launches(path):
    txt = open(path).read()
    start = txt.find('"ID"')
    rows = list(csv.DictReader(io.StringIO(txt[start:])))
    agg = {}
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        k = r["Kernel Name"].split("(")[0]
        t = float(r["Metric Value"].replace(",", ""))
        a = agg.setdefault(k, {"count": 0, "time": 0.0, "unit": r["Metric Unit"]})
        a["count"] += 1
        a["time"] += t
    tot = sum(a["time"] for a in agg.values()) or 1.0
    for a in agg.values():
        a["share"] = a["time"] / tot
    return agg


if __name__ == "__main__":
    rep, csvp, out = sys.argv[1], sys.argv[2], sys.argv[3]
    systems = int(sys.argv[4]) if len(sys.argv) > 4 else 4096
    s = {"report": rep, "full": raw(rep), "launch_list": launches(csvp)}
    f = s["full"]
    def num(k):
        x = f[k]["value"].replace(",", "")
        u = f[k]["unit"]
        mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}.get(u, 1)
        return float(x) * mult
    s["dram_bytes_per_launch"] = num("dram_read") + num("dram_write")
    s["systems_per_launch"] = systems
    json.dump(s, open(out, "w"), indent=1)
    print(json.dumps({k: s[k] for k in ("dram_bytes_per_launch", "systems_per_launch")}))
