"""Summarise `ncu --set full` reports (profiles/README_r02.md) into the committed JSON, and regenerate
profiles/traffic.json (DRAM bytes per launch read by bench.py for roofline.traffic).

    python profiles/ncu_summary.py OUT.json REPORT.ncu-rep [REPORT ...]
    python profiles/ncu_summary.py --traffic OUT.json   # rebuild traffic.json from the summary OUT.json

Per kernel launch: duration, DRAM read/write bytes, L2 hit rate, L1TEX global-load wavefronts (the
random-gather limit), issue activity, achieved occupancy, registers, the top stall reasons."""
import csv
import json
import subprocess
import sys

METRICS = {
    "gpu__time_duration.sum": "duration_us",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "lts__t_sector_hit_rate.pct": "l2_hit_pct",
    "l1tex__data_pipe_lsu_wavefronts_mem_lgds.sum": "l1tex_lgds_wavefronts",
    "l1tex__t_sectors_pipe_lsu_mem_global_op_ldgsts.sum": "ldgsts_sectors",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active_pct",
    "launch__registers_per_thread": "registers",
    "launch__grid_size": "grid",
    "smsp__inst_executed.sum": "warp_instructions",
}
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "us": 1, "ms": 1e3, "ns": 1e-3, "usecond": 1,
        "msecond": 1e3, "nsecond": 1e-3}


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, u = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[h.index("Kernel Name")], "report": rep.split("/")[-1]}
        for m, key in METRICS.items():
            if m in h:
                i = h.index(m)
                try:
                    v = float(r[i].replace(",", ""))
                except ValueError:
                    continue
                d[key] = v * UNIT.get(u[i], 1)
        res.append(d)
    return res


def stalls(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    secs, cur = [], None
    for r in rows:
        if r and r[0] == "Kernel Name":
            cur = {"name": r[1], "rows": []}
            secs.append(cur)
        elif cur is not None:
            cur["rows"].append(r)
    res = []
    for sec in secs:
        rs = sec["rows"]
        h = rs[0]
        body = [r for r in rs[1:] if len(r) == len(h) and r[0] != "Address"]
        names = [n for n in h if n.startswith("stall_") and "Not Issued" not in n]
        agg = {n[6:]: sum(float(r[h.index(n)] or 0) for r in body) for n in names}
        tot = sum(agg.values()) or 1.0
        res.append((sec["name"], sorted(((round(100 * v / tot, 1), k) for k, v in agg.items()), reverse=True)[:5]))
    return res


def main():
    if sys.argv[1] == "--traffic":
        summ = json.load(open(sys.argv[2]))
        cls = {"k_dual_rb": "pdhg_dual", "k_primal_rb": "pdhg_primal", "k_primal_push": "pdhg_primal_col",
               "k_feas_rb": "feas", "k_sample": "sample"}
        out = {"_source": f"profiles/ncu_summary.py --traffic {sys.argv[2]} (dram read + write bytes per launch, "
                          "ncu --set full --clock-control none, cold caches)", "config5_fp32": {}}
        for d in summ["launches"]:
            for k, c in cls.items():
                if f"{k}<" in d["kernel"] or d["kernel"].startswith(k + "("):
                    out["config5_fp32"].setdefault(c, int(d.get("dram_read", 0) + d.get("dram_write", 0)))
        json.dump(out, open("profiles/traffic.json", "w"), indent=1)
        print(json.dumps(out, indent=1))
        return
    launches = []
    for rep in sys.argv[2:]:
        ls = raw(rep)
        st = stalls(rep)  # [(function name, top stalls)] per source-page section
        # the source page groups its sections by function: pair them with the launches of the same
        # function, in order
        by_fn = {}
        for name, top in st:
            by_fn.setdefault(name, []).append(top)
        for d in ls:
            base = d["kernel"].split("(")[0].replace("void ", "").split("<")[0].split("::")[-1]
            for name, tops in by_fn.items():
                if tops and name.split("(")[0].replace("void ", "").split("<")[0].split("::")[-1] == base:
                    d["top_stalls_pct"] = tops.pop(0)
                    break
            launches.append(d)
    json.dump({"launches": launches}, open(sys.argv[1], "w"), indent=1)
    for d in launches:
        print(d["kernel"][:60], round(d.get("duration_us", 0), 1), "us", "DRAM", round((d.get("dram_read", 0) + d.get("dram_write", 0)) / 1e6, 1), "MB")


if __name__ == "__main__":
    main()
