"""Summarize an ncu --set full report of bench.py's step into profiles/<round>/:
per-launch metrics JSON, and profiles/k2_traffic.json (DRAM bytes per K2 launch, averaged
over the step's K2 launches -- the `traffic` field of bench.py's roofline object).

    python tools/summarize_ncu.py gpurun_out/prof_r01.ncu-rep profiles/r01
"""
import csv, io, json, os, subprocess, sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402

rep, outdir = sys.argv[1], sys.argv[2]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
keys = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sectors.sum.pct_of_peak_sustained_elapsed",
        "l1tex__m_xbar2l1tex_read_bytes.sum", "launch__grid_size", "launch__registers_per_thread",
        "sm__cycles_elapsed.avg.per_second"]
keys = [k for k in keys if k in hdr]
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
launches = []
for r in rows[2:]:
    d = {}
    for k in keys:
        v = r[hdr.index(k)]
        u = units[hdr.index(k)]
        if k == "Kernel Name":
            d[k] = v
        elif u in scale:
            d[k.replace(".sum", "_bytes")] = float(v) * scale[u]
        else:
            d[k] = float(v)
    launches.append(d)
layers = synth.flux_double_block(1) + synth.flux_single_block(1)
by = {L.name: L for L in layers}
# the step's launch groups (bench.flux_step_grouped): img + txt of each double-block kind, then the single block
groups = [[by[f"double_{s_}_{k}"] for s_ in ("img", "txt")] for k in ("qkv", "proj", "mlp_up", "mlp_down")]
groups += [[by["single_linear1"]], [by["single_linear2"]]]
k2 = [d for d in launches if "k2_" in d["Kernel Name"]]
k1 = [d for d in launches if "k1_" in d["Kernel Name"]]
if len(k2) == len(layers):                       # serial form (one launch per linear)
    groups = [[L] for L in layers]
alg = []
for grp, d, d1 in zip(groups, k2, k1):
    alg_bytes = sum(0.5625 * (L.M + L.N) * L.K + 2 * (L.M + L.N) * L.r + 2 * L.N + 2 * L.M * L.N for L in grp)
    k1_bytes = sum(L.M * L.K * 2.5625 + 2 * L.M * L.r for L in grp)
    d["layer"] = "+".join(L.name for L in grp)
    d["algorithmic_min_bytes"] = alg_bytes
    d["algorithmic_flops"] = sum(2.0 * L.M * L.N * L.K for L in grp)
    d["tflops_under_ncu"] = d["algorithmic_flops"] / (d["gpu__time_duration.sum"] * 1e-6) / 1e12
    d1["layer"] = d["layer"]
    d1["algorithmic_bytes"] = k1_bytes
    d1["tbs_under_ncu"] = k1_bytes / (d1["gpu__time_duration.sum"] * 1e-6) / 1e12
    alg.append(alg_bytes)
traffic = [d["dram__bytes_read_bytes"] + d["dram__bytes_write_bytes"] for d in k2]
summary = {
    "source": os.path.basename(rep),
    "note": "ncu --set full --clock-control none; one grouped bench step (tools/step_once.py: 6 K1 + 6 K2 launches). "
            "Per-launch times are cold-cache and serialised: compare shares, not absolutes.",
    "k2_traffic_bytes_per_launch_mean": sum(traffic) / max(1, len(traffic)),
    "k2_algorithmic_min_bytes_per_launch_mean": sum(alg) / max(1, len(alg)),
    "k2_time_share": sum(d["gpu__time_duration.sum"] for d in k2) / sum(d["gpu__time_duration.sum"] for d in launches),
    "launches": launches,
}
os.makedirs(outdir, exist_ok=True)
json.dump(summary, open(os.path.join(outdir, "ncu_full_summary.json"), "w"), indent=1)
json.dump({"bytes_per_launch": round(summary["k2_traffic_bytes_per_launch_mean"]),
           "algorithmic_min_bytes_per_launch": round(summary["k2_algorithmic_min_bytes_per_launch_mean"]),
           "source": f"{outdir}/ncu_full_summary.json",
           "definition": "mean over the step's K2 launches of dram__bytes_read.sum + dram__bytes_write.sum"},
          open(os.path.join(os.path.dirname(outdir.rstrip('/')), "k2_traffic.json"), "w"), indent=1)
print(json.dumps({k: v for k, v in summary.items() if k != "launches"}, indent=1))
for d in k2:
    print(f"K2 {d["layer"]:40s} {d['gpu__time_duration.sum']:8.1f} us  tensor {d.get('sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active', 0):5.1f}%  "
          f"dram {(d['dram__bytes_read_bytes'] + d['dram__bytes_write_bytes'])/1e6:7.1f} MB  alg {d['algorithmic_min_bytes']/1e6:7.1f} MB")
for d in k1:
    print(f"K1 {d.get('layer', '?'):40s} {d['gpu__time_duration.sum']:8.1f} us  dram {(d['dram__bytes_read_bytes'] + d['dram__bytes_write_bytes'])/1e6:7.1f} MB  "
          f"alg {d.get('algorithmic_bytes', 0)/1e6:7.1f} MB  {d.get('tbs_under_ncu', 0):.2f} TB/s")
