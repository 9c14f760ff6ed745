"""Summarise an ncu --set full capture of the fused kernel into profiles/.

    python tools/ncu_summary.py gpurun_out/prof_flux.ncu-rep profiles/ncu_r01_<tag> [plan_flops]

Writes <out>.json (key counters per launch) and <out>_stalls.txt (top SASS
stall sites) — the evidence behind bench.py's roofline block."""
import csv
import io
import json
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.per_cycle_active", "launch__registers_per_thread",
        "sm__cycles_elapsed.avg.per_second", "lts__t_sector_hit_rate.pct",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "launch__grid_size", "launch__block_size",
        "smsp__inst_executed.sum", "launch__shared_mem_per_block_dynamic",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__m_xbar2l1tex_read_bytes.sum"]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    launches = []
    for vals in rows[2:]:
        d = {"kernel": vals[hdr.index("Kernel Name")]}
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                d[k] = {"value": vals[i], "unit": units[i]}
        launches.append(d)
    return launches


def stalls(rep, top=30):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[1]
    data = rows[2:]
    ia, isrc = hdr.index("Address"), hdr.index("Source")
    ist, iex = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
    tot = sum(float(r[ist] or 0) for r in data) or 1.0
    lines = [f"total stall samples {tot:.0f}"]
    for r in sorted(data, key=lambda r: -float(r[ist] or 0))[:top]:
        lines.append(f"{float(r[ist]) / tot * 100:5.1f}%  {r[isrc].strip()[:100]}  (executed {r[iex]})")
    return "\n".join(lines)


def main():
    rep, out = sys.argv[1], sys.argv[2]
    plan_flops = float(sys.argv[3]) if len(sys.argv) > 3 else None
    ls = raw(rep)
    summary = {"report": rep, "launches": ls}
    if ls and plan_flops:
        t = float(ls[0]["gpu__time_duration.sum"]["value"])
        unit = ls[0]["gpu__time_duration.sum"]["unit"]
        sec = t * {"ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3}.get(unit, 1e-9)
        summary["achieved_tflops_under_ncu"] = plan_flops / sec / 1e12
    if ls:
        def mb(k):
            v = ls[0].get(k)
            if not v:
                return None
            s = float(v["value"])
            return s * {"Mbyte": 1e6, "Gbyte": 1e9, "Kbyte": 1e3, "byte": 1.0}.get(v["unit"], 1.0)
        rd, wr = mb("dram__bytes_read.sum"), mb("dram__bytes_write.sum")
        if rd is not None and wr is not None:
            summary["dram_bytes_per_launch"] = rd + wr
    with open(out + ".json", "w") as f:
        json.dump(summary, f, indent=1)
    with open(out + "_stalls.txt", "w") as f:
        f.write(stalls(rep))
    print(json.dumps({k: v for k, v in summary.items() if k != "launches"}, indent=1))


if __name__ == "__main__":
    main()
