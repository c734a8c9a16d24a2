"""Summarise an `ncu --set full` report for profiles/: per kernel the
duration, DRAM bytes / throughput, SM throughput, occupancy and registers;
also writes profiles/ncu_traffic.json (kernel -> DRAM bytes per launch) that
bench.py reports as roofline.traffic.

usage: python scripts/ncu_summarize.py REPORT.ncu-rep OUT_SUMMARY.txt [TRAFFIC.json]
"""
import csv
import json
import subprocess
import sys
from collections import defaultdict

METRICS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__inst_executed.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread",
    "launch__grid_size",
    "launch__block_size",
    "lts__t_sector_hit_rate.pct",
]


WIDTH = {"unsigned char": "u8", "unsigned short": "u16", "unsigned int": "u32", "Contig8Src": "u8"}


def short(name):
    """ncu kernel name -> the name bench.py's per-launch timing uses."""
    name = name.replace("scz::", "").replace("(anonymous namespace)::", "").replace("<unnamed>::", "")
    name = name.replace("void ", "")
    base = name.split("(")[0]
    stem = base.split("<")[0]
    targs = base[len(stem) + 1:-1] if "<" in base else ""
    width = None
    for key, w in WIDTH.items():
        if targs.startswith(key) or targs.startswith("SplitSrc<" + key):
            width = w
            break
    if stem in ("k_rows_small", "k_rows_fast"):
        stem = "k_rows_out"
    if stem == "k_rows_small8":  # u8 only
        return "k_rows_out/u8"
    if stem == "k_rans_enc_v2_u8u16":
        return "k_rans_enc_v2/u8u16"
    if stem == "k_materialize_u8u16":
        return "k_materialize"
    if stem == "k_rowhist2":
        stem = "k_rowhist"
    if stem in ("k_rans_enc_v2", "k_rans_dec_v2", "k_rans_enc_v1", "k_rans_dec_v1", "k_materialize",
                "k_row_sums", "k_rows_out") and width:
        return f"{stem}/{width}"
    return stem


def main():
    rep, out = sys.argv[1], sys.argv[2]
    traffic_path = sys.argv[3] if len(sys.argv) > 3 else None
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", ",".join(METRICS)],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    hdr = rows[0]
    ik = hdr.index("Kernel Name")
    col = {m: hdr.index(m) for m in METRICS if m in hdr}
    units = rows[1]
    scale = {"ns": 1.0, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6, "s": 1e9, "second": 1e9,
             "nsecond": 1.0, "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
    agg = defaultdict(list)
    for r in rows[2:]:
        if len(r) < len(hdr):
            continue
        vals = {}
        for m, j in col.items():
            try:
                vals[m] = float(r[j].replace(",", "")) * scale.get(units[j], 1.0)
            except ValueError:
                vals[m] = float("nan")
        agg[short(r[ik])].append(vals)
    lines = [f"# ncu --set full summary of {rep.split('/')[-1]} (per-launch means; cold caches, serialised)", ""]
    traffic = {}
    for k, vs in agg.items():
        mean = {m: sum(v[m] for v in vs) / len(vs) for m in col}
        dram = mean.get("dram__bytes_read.sum", 0) + mean.get("dram__bytes_write.sum", 0)
        dur = mean.get("gpu__time_duration.sum", float("nan"))  # ns
        traffic[k] = dram
        lines += [
            f"## {k}  ({len(vs)} launches)",
            f"    duration            {dur / 1e3:10.2f} us",
            f"    dram read + write   {dram / 1e6:10.2f} MB   ({dram / dur:.0f} GB/s achieved)" if dur == dur and dur else "",
            f"    dram throughput     {mean.get('gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed', 0):10.1f} % of peak",
            f"    SM throughput       {mean.get('sm__throughput.avg.pct_of_peak_sustained_elapsed', 0):10.1f} %",
            f"    issue active        {mean.get('smsp__issue_active.avg.pct_of_peak_sustained_active', 0):10.1f} %",
            f"    warps active        {mean.get('sm__warps_active.avg.pct_of_peak_sustained_active', 0):10.1f} % of max",
            f"    L2 hit rate         {mean.get('lts__t_sector_hit_rate.pct', 0):10.1f} %",
            f"    warp instructions   {mean.get('smsp__inst_executed.sum', 0):10.3g}",
            f"    smem bank conflicts {mean.get('l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum', 0):10.3g}",
            f"    registers / thread  {mean.get('launch__registers_per_thread', 0):10.0f}",
            f"    grid x block        {mean.get('launch__grid_size', 0):10.0f} x {mean.get('launch__block_size', 0):.0f}",
            "",
        ]
    open(out, "w").write("\n".join(l for l in lines if l is not None) + "\n")
    if traffic_path:
        json.dump(traffic, open(traffic_path, "w"), indent=1, sort_keys=True)
    print(open(out).read())


if __name__ == "__main__":
    main()
