"""Turn ncu outputs into the committed profile summaries under profiles/.

    python tools/ncu_summary.py <tag> <launches.csv> <full.ncu-rep> [config]

Writes
  profiles/<tag>_launches.csv          every launch: kernel, grid, block, ns
  profiles/<tag>_launch_summary.md     per kernel: launches, total / mean us, share
  profiles/<tag>_ncu_full_summary.csv  --set full metrics of the captured kernels
  profiles/ncu_traffic.json            dram read+write bytes per launch, keyed by
                                       the bench's traced-kernel names (roofline.traffic)
"""
import csv
import io
import json
import subprocess
import sys
from collections import defaultdict
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
PROF = ROOT / "profiles"

# bench / LeoTrace kernel names -> C kernel symbol prefixes
TRACE_TO_KERNEL = {
    "sync_trace": ("k_sync_wc_smem", "k_sync<false>"),
    "reach_fast": ("k_reach_unit", "k_reach_fast"),
    "prune_edges": ("k_prune_edges_smem", "k_prune_edges"),
    "blame_count": ("k_blame<0>",),
    "blame_fill": ("k_blame<1>",),
    "bin_samples": ("k_bin_hash", "k_bin_count", "k_bin_samples"),
    "block_walk": ("k_block_walk",),
    "slice": ("k_slice",),
    "segsort_unique": ("segsort_unique_u64",),
}


def short(name: str) -> str:
    n = name.replace("void ", "")
    n = n.split("(")[0]
    return n.replace("leo::", "")


def launches(path: Path):
    rows = []
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    rd = csv.DictReader(io.StringIO("".join(lines)))
    for r in rd:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        rows.append((short(r["Kernel Name"]), r["Grid Size"], r["Block Size"], float(r["Metric Value"])))
    return rows


def full_metrics(rep: Path):
    """--set full metrics from an .ncu-rep or its exported raw page (.csv)."""
    if str(rep).endswith(".csv"):
        out = Path(rep).read_text()
    else:
        out = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True,
                             text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[0]
    want = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "lts__t_bytes.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
            "smsp__thread_inst_executed_per_inst_executed.ratio", "launch__grid_size",
            "launch__block_size", "launch__shared_mem_per_block_dynamic", "launch__registers_per_thread",
            "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum",
            "smsp__inst_executed.sum", "sm__cycles_active.avg", "smsp__cycles_active.max",
            "smsp__issue_active.avg.pct_of_peak_sustained_active",
            "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"]
    units = rows[1]
    idx = [h.index(w) for w in want if w in h]
    recs = []
    for r in rows[2:]:
        d = {h[i]: r[i] for i in idx}
        d["_units"] = {h[i]: units[i] for i in idx}
        recs.append(d)
    return recs, [h[i] for i in idx]


def to_bytes(v: str, unit: str) -> float:
    x = float(v.replace(",", ""))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}
    return x * scale.get(unit, 1)


def main():
    tag, lpath, rep = sys.argv[1], Path(sys.argv[2]), Path(sys.argv[3])
    config = sys.argv[4] if len(sys.argv) > 4 else "c2"
    PROF.mkdir(exist_ok=True)
    L = launches(lpath)
    with open(PROF / f"{tag}_launches.csv", "w") as f:
        f.write("kernel,grid,block,ns\n")
        for k, g, b, ns in L:
            f.write(f"\"{k}\",\"{g}\",\"{b}\",{ns:.0f}\n")
    agg = defaultdict(lambda: [0, 0.0])
    for k, _, _, ns in L:
        if k.startswith("at::") or "elementwise" in k or "Fill" in k:
            continue
        agg[k][0] += 1
        agg[k][1] += ns
    tot = sum(v[1] for v in agg.values())
    with open(PROF / f"{tag}_launch_summary.md", "w") as f:
        f.write(f"# ncu launch list ({lpath.name}): libleo_b200 kernels only\n\n")
        f.write("Cold-cache, serialised per-launch times (ncu --metrics gpu__time_duration.sum "
                "--clock-control none); compare shares, not absolutes.\n\n")
        f.write("| kernel | launches | total us | mean us | share |\n|---|---|---|---|---|\n")
        for k, (n, ns) in sorted(agg.items(), key=lambda x: -x[1][1]):
            f.write(f"| {k} | {n} | {ns / 1e3:.1f} | {ns / n / 1e3:.2f} | {100 * ns / tot:.1f}% |\n")
    recs, cols = full_metrics(rep)
    with open(PROF / f"{tag}_ncu_full_summary.csv", "w") as f:
        w = csv.writer(f)
        w.writerow(cols)
        w.writerow([recs[0]["_units"].get(c, "") for c in cols] if recs else [])
        for d in recs:
            w.writerow([d.get(c, "") for c in cols])
    traffic_path = PROF / "ncu_traffic.json"
    traffic = json.loads(traffic_path.read_text()) if traffic_path.exists() else {}
    tc = traffic.setdefault(config, {})
    for trace, syms in TRACE_TO_KERNEL.items():
        for d in recs:
            name = short(d["Kernel Name"])
            if any(name.startswith(s) for s in syms):
                u = d["_units"]
                rd = to_bytes(d["dram__bytes_read.sum"], u["dram__bytes_read.sum"])
                wr = to_bytes(d["dram__bytes_write.sum"], u["dram__bytes_write.sum"])
                tc[trace] = int(rd + wr)
                break
    traffic_path.write_text(json.dumps(traffic, indent=1, sort_keys=True) + "\n")
    # per traced kernel: DRAM bytes, global-load sectors per request, warps active
    stats_path = PROF / "ncu_kernel_stats.json"
    stats = json.loads(stats_path.read_text()) if stats_path.exists() else {}
    sc = stats.setdefault(config, {})
    for trace, syms in TRACE_TO_KERNEL.items():
        for d in recs:
            name = short(d["Kernel Name"])
            if any(name.startswith(sy) for sy in syms):
                u = d["_units"]
                sec = float(d.get("l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", "0").replace(",", "") or 0)
                req = float(d.get("l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum", "0").replace(",", "") or 0)
                sc[trace] = {"kernel": name, "dram_bytes": tc.get(trace),
                             "sectors_per_request": round(sec / req, 2) if req else None,
                             "warps_active_pct": float(d.get("sm__warps_active.avg.pct_of_peak_sustained_active", "0") or 0),
                             "us": float(d.get("gpu__time_duration.sum", "0").replace(",", "") or 0)
                             * {"msecond": 1e3, "usecond": 1.0, "nsecond": 1e-3}.get(
                                 u.get("gpu__time_duration.sum", "usecond"), 1.0)}
                break
    stats_path.write_text(json.dumps(stats, indent=1, sort_keys=True) + "\n")
    print(f"wrote {tag}: {len(L)} launches, {len(recs)} full captures; traffic {tc}")


if __name__ == "__main__":
    main()
