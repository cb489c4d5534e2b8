"""Summarise ncu captures for profiles/ (committed evidence).

Usage: python scripts/profile_summary.py <full.ncu-rep> <launches.csv|-> <out_prefix> [config] [pipes.csv]
Writes <out_prefix>_launches.txt (kernel launch list with durations) and
<out_prefix>_band_kernel.txt (speed-of-light, memory traffic, occupancy,
stall reasons and per-phase instruction split of the dominant kernel), and
updates profiles/traffic.json with the kernel's measured DRAM bytes/launch.
"""
import csv
import io
import json
import os
import subprocess
import sys

rep, launches, prefix = sys.argv[1], sys.argv[2], sys.argv[3]


def is_band(name):
    """The generator kernels: band_kernel<PSF> and band_sorted_kernel (not sample_band_kernel)."""
    return "band_kernel" in name and "sample_band" not in name or "band_sorted_kernel" in name
cfgname = sys.argv[4] if len(sys.argv) > 4 else "c2"
pipes_csv = sys.argv[5] if len(sys.argv) > 5 else None
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def band_ranges():
    """Source regions of band.cuh located by their section comments."""
    src = open(os.path.join(root, "paper_2512_09664_b200", "csrc", "band.cuh")).read().split("\n")
    marks = [("prologue", "// Per-pair prologue"), ("splat", "// Tight window of one particle-frame"),
             ("store", "// Epilogue: one output quad"), ("stage", "// Range of seeding cells"),
             ("gen", "// One regenerated particle"), ("loop", "// Worker warps: regenerate"),
             ("sorted", "// Bank-sorted splat for large windows"),
             ("kernel", "// Workers: particles of the staged item"),
             ("end", "// Particle arrays of the generator")]
    pos = []
    for name, m in marks:
        ln = next(i + 1 for i, l in enumerate(src) if l.startswith(m))
        pos.append((name, ln))
    pos.sort(key=lambda t: t[1])
    out = []
    for (n, a), (_, b) in zip(pos, pos[1:]):
        if n != "end":
            out.append(f"{n}=band.cuh:{a}-{b - 1}")
    return ",".join(out + ["fused_helpers=fused.cuh:1-1200", "philox=common.cuh:1-400"])


# ---- launch list
rows = [r for r in csv.DictReader(l for l in open(launches) if not l.startswith("=="))] if launches != "-" else []
with open(prefix + "_launches.txt", "w") if rows else open(os.devnull, "w") as fh:
    fh.write("# ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised)\n")
    fh.write(f"# command: python bench.py --steps 5 --warmup 3 --no-cpu-baseline --config {cfgname}\n")
    for r in rows:
        fh.write(f"{r['ID']:>4s}  {r['Kernel Name'][:70]:70s}  {float(r['Metric Value'])/1000:9.2f} us\n")
    band = [float(r["Metric Value"]) for r in rows if is_band(r["Kernel Name"])]
    other = [float(r["Metric Value"]) for r in rows if not is_band(r["Kernel Name"])]
    if band:
        fh.write(f"# band_kernel launches: {len(band)}, mean {sum(band)/len(band)/1000:.2f} us; "
                 f"other kernels (bench L2 flush): {len(other)}\n")

def pipes_section(path, alg_bytes):
    """Pipe utilisation / shared atomics / occupancy of each band-kernel launch
    (scripts/profile_run.sh metrics pass) and its DRAM write traffic including
    the dirty lines the following L2-flush kernel evicts."""
    rows = [r for r in csv.DictReader(l for l in open(path) if not l.startswith("=="))]
    launches = []
    for r in rows:
        key = (r["ID"], r["Kernel Name"])
        if not launches or launches[-1]["key"] != key:
            launches.append({"key": key, "name": r["Kernel Name"], "m": {}})
        try:
            v = float(r["Metric Value"].replace(",", ""))
        except ValueError:
            continue
        u = r.get("Metric Unit", "")
        v *= {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "usecond": 1e3, "msecond": 1e6}.get(u, 1)
        launches[-1]["m"][r["Metric Name"]] = v
    out = ["\n# pipes / shared atomics / DRAM per band-kernel launch (ncu --metrics, scripts/profile_run.sh)\n"]
    flush_bytes = 256 * 1024 * 1024
    for i, L in enumerate(launches):
        if not is_band(L["name"]):
            continue
        m = L["m"]
        nxt = launches[i + 1]["m"] if i + 1 < len(launches) else {}
        spill = max(0.0, nxt.get("dram__bytes_write.sum", 0.0) - flush_bytes) if nxt else float("nan")
        out.append(f"launch {L['key'][0]}: {m.get('gpu__time_duration.sum', float('nan'))/1e3:.2f} us\n")
        for k in ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
                  "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
                  "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active",
                  "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
                  "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
                  "sm__warps_active.avg.pct_of_peak_sustained_active",
                  "sm__inst_executed.avg.per_cycle_active", "sm__inst_executed.sum",
                  "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum",
                  "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_atom.sum",
                  "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
                  "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
                  "dram__bytes_read.sum", "dram__bytes_write.sum"):
            out.append(f"  {k:78s} {m.get(k, float('nan')):.4g}\n")
        atom = m.get("l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum", 0.0)
        conf = m.get("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_atom.sum", 0.0)
        if atom:
            out.append(f"  shared-atomic wavefronts that are bank conflicts: {100*conf/atom:.1f}%\n")
        if spill == spill:
            tot = m.get("dram__bytes_write.sum", 0.0) + spill
            out.append(f"  DRAM write incl. dirty lines evicted by the next flush: {tot:.4g} B "
                       f"(algorithmic {alg_bytes} B, ratio {tot/alg_bytes:.3f})\n")
    return "".join(out)


# ---- full capture
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(raw)))
hdr, units, vals = r[0], r[1], r[2]
d = dict(zip(hdr, vals))
un = dict(zip(hdr, units))
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1, "usecond": 1e3,
         "msecond": 1e6, "second": 1e9, "ns": 1, "us": 1e3, "ms": 1e6}


def f(k):
    # bytes for byte metrics, nanoseconds for time metrics, raw otherwise
    try:
        return float(d[k]) * SCALE.get(un.get(k, ""), 1)
    except (KeyError, ValueError):
        return float("nan")


dram_r, dram_w = f("dram__bytes_read.sum"), f("dram__bytes_write.sum")
dur_ns = f("gpu__time_duration.sum")
stalls = {k[len("smsp__pcsamp_warps_issue_stalled_"):]: f(k) for k in hdr
          if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")}
tot = sum(v for v in stalls.values() if v == v) or 1.0
phases = subprocess.run([sys.executable, os.path.join(root, "scripts", "ncu_lines.py"), rep, "0",
                         band_ranges()],
                        capture_output=True, text=True).stdout
with open(prefix + "_band_kernel.txt", "w") as fh:
    fh.write("# ncu --set full --clock-control none --import-source on -k regex:'band_(sorted_)?kernel' -s 3 -c 1\n")
    fh.write(f"#   python bench.py --steps 3 --warmup 3 --no-cpu-baseline --config {cfgname}\n")
    fh.write(f"duration_us                {dur_ns/1000:.2f}\n")
    fh.write(f"dram_bytes_read            {dram_r:.0f}\n")
    fh.write(f"dram_bytes_write           {dram_w:.0f}\n")
    sys.path.insert(0, root)
    import bench  # noqa: E402
    H, W, B = bench.CONFIGS[cfgname][:3]
    fh.write(f"algorithmic_bytes          {B*2*H*W*4} (2 f32 frames x {B} pairs of {H}x{W})\n")
    for k in ["sm__throughput.avg.pct_of_peak_sustained_elapsed",
              "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
              "dram__throughput.avg.pct_of_peak_sustained_elapsed",
              "smsp__inst_executed.sum", "sm__inst_executed.avg.per_cycle_active",
              "sm__warps_active.avg.pct_of_peak_sustained_active",
              "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic",
              "launch__grid_size", "launch__block_size", "launch__occupancy_limit_registers",
              "launch__occupancy_limit_shared_mem"]:
        fh.write(f"{k:60s} {d.get(k, 'n/a')}\n")
    fh.write("\n# warp stall samples (% of all)\n")
    for k, v in sorted(stalls.items(), key=lambda kv: -kv[1])[:12]:
        fh.write(f"  {k:30s} {100*v/tot:5.1f}\n")
    fh.write("\n# instruction / stall-sample split by source region (scripts/ncu_lines.py)\n")
    fh.write(phases)
    if pipes_csv:
        fh.write(pipes_section(pipes_csv, B * 2 * H * W * 4))

tp = os.path.join(root, "profiles", "traffic.json")
tj = json.load(open(tp)) if os.path.exists(tp) else {}
tj[cfgname] = {"kernel": "pgb::band_sorted_kernel" if cfgname == "c3" else "pgb::band_kernel<0>", "dram_bytes_per_launch": dram_r + dram_w,
            "dram_read": dram_r, "dram_write": dram_w, "duration_us_ncu": dur_ns / 1000,
            "source": os.path.basename(prefix) + "_band_kernel.txt"}
json.dump(tj, open(tp, "w"), indent=1)
print(open(prefix + "_band_kernel.txt").read())
