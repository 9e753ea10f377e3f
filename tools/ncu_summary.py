"""Summarise an ncu --set full capture of the window kernel into
profiles/ncu_summary.json (read by bench.py for roofline.traffic).

    python tools/ncu_summary.py REPORT.ncu-rep PLAIN_WINDOW_COUNTS.log OUT.json [SOURCE_SHA]

SOURCE_SHA is the sha256 of the kernel source (csrc/persist.cu) the capture
ran; bench.py uses the traffic figure only while the source still matches."""
import csv, hashlib, io, json, os, subprocess, sys
rep, plain, out = sys.argv[1], sys.argv[2], sys.argv[3]
src_sha = sys.argv[4] if len(sys.argv) > 4 else hashlib.sha256(open(os.path.join(
    os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
    "paper_2006_14602_b200", "csrc", "persist.cu"), "rb").read()).hexdigest()
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, vals = rows[0], rows[1], rows[2]
def get(name):
    return float(vals[hdr.index(name)].replace(",", "")) if name in hdr else None
def unit(name):
    return units[hdr.index(name)] if name in hdr else None
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
tscale = {"ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "s": 1.0, "second": 1.0}
rd = get("dram__bytes_read.sum") * scale[unit("dram__bytes_read.sum")]
wr = get("dram__bytes_write.sum") * scale[unit("dram__bytes_write.sum")]
t = get("gpu__time_duration.sum") * tscale[unit("gpu__time_duration.sum")]
wins = [json.loads(l) for l in open(plain) if l.startswith("{")]
last = wins[-1]
summ = {
    "kernel": "k_windowP (persistent window kernel), one window under ncu --set full",
    "report": rep, "window_index": last["window"],
    "duration_s_under_ncu": t,
    "dram_read_bytes": rd, "dram_write_bytes": wr, "dram_bytes": rd + wr,
    "node_updates": last["node_updates"], "algo_bytes": last["algo_bytes"],
    "stage_traffic_bytes_per_node": (rd + wr) / last["node_updates"],
    "algo_bytes_per_node": last["algo_bytes"] / last["node_updates"],
    "dram_throughput_pct": get("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
    "sm_throughput_pct": get("sm__throughput.avg.pct_of_peak_sustained_elapsed"),
    "issue_active_pct": get("smsp__issue_active.avg.pct_of_peak_sustained_active"),
    "warps_active_pct": get("sm__warps_active.avg.pct_of_peak_sustained_active"),
    "fp64_pipe_pct": get("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active"),
    "registers_per_thread": get("launch__registers_per_thread"),
    "note": "ncu replays serialize and run cold-cache; compare shares, not absolute time",
    "persist_cu_sha256": src_sha,
}
json.dump(summ, open(out, "w"), indent=1)
print(json.dumps(summ, indent=1))
