"""Summarise an ncu report (or a launch-list CSV) into the plain-text files kept under profiles/.

    python tools/ncu_summary.py full  <report.ncu-rep | raw.csv> <out.txt> [evals_per_launch]
    python tools/ncu_summary.py list  <launches.csv>   <out.txt>
"""
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed", "l1tex__data_pipe_lsu_wavefronts.sum",
        "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum", "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum",
        "l1tex__t_sector_hit_rate.pct", "lts__t_sectors_srcunit_tex_op_read.sum", "lts__t_sector_hit_rate.pct",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "sm__inst_executed.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "launch__occupancy_limit_registers", "sm__cycles_elapsed.avg.per_second",
        "smsp__thread_inst_executed_per_inst_executed.ratio"]

SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def _num(s):
    return float(s.replace(",", ""))


def full(rep, out, evals=None):
    if rep.endswith(".csv"):  # `ncu -i <rep> --page raw --csv` already exported on the GPU box
        raw = open(rep).read()
    else:
        raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    lines = [f"ncu --set full summary of {rep}"]
    for vals in rows[2:]:
        d = {h: (u, v) for h, u, v in zip(hdr, units, vals)}
        lines.append(f"\nkernel: {d.get('Kernel Name', ('', '?'))[1]}")
        for k in KEYS:
            if k in d:
                lines.append(f"  {k:75s} {d[k][1]:>22s} {d[k][0]}")
        if evals:
            if "l1tex__data_pipe_lsu_wavefronts.sum" in d:
                wf = _num(d["l1tex__data_pipe_lsu_wavefronts.sum"][1])
            else:
                key = [k for k in d if k.endswith("l1tex__data_pipe_lsu_wavefronts.avg")][0]
                if d[key][1] != "no data":
                    wf = _num(d[key][1]) * 148
                else:  # only the utilisation was captured: 1 wavefront per SM per cycle at 100 %
                    pct = _num(d["l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed"][1]) / 100
                    t_ms = _num(d["gpu__time_duration.sum"][1])
                    ghz = _num(d["sm__cycles_elapsed.avg.per_second"][1])
                    wf = pct * t_ms * 1e-3 * ghz * 1e9 * 148
            lines.append(f"  l1tex__data_pipe_lsu_wavefronts (sum over 148 SMs) {wf:.4g}")
            rd = _num(d["dram__bytes_read.sum"][1]) * SCALE.get(d["dram__bytes_read.sum"][0], 1.0)
            wr = _num(d["dram__bytes_write.sum"][1]) * SCALE.get(d["dram__bytes_write.sum"][0], 1.0)
            lines.append(f"  derived: evals/launch {evals:.4g}; L1 wavefronts/eval {wf / evals:.2f}; "
                         f"DRAM bytes/eval {(rd + wr) / evals:.3f} (read+write {rd + wr:.4g} B/launch)")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


def launch_list(path, out):
    txt = open(path).read()
    start = txt.find('"ID"')
    rows = list(csv.DictReader(io.StringIO(txt[start:])))
    agg = {}
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"].split("(")[0]
        v = _num(r["Metric Value"])
        scale = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0,
                 "second": 1e3, "s": 1e3}.get(r.get("Metric Unit", "nsecond"), 1e-6)
        agg.setdefault(name, [0, 0.0])
        agg[name][0] += 1
        agg[name][1] += v * scale
    total = sum(v[1] for v in agg.values())
    lines = [f"ncu launch list ({path}): {sum(v[0] for v in agg.values())} launches, {total:.2f} ms total "
             f"(serialised, cold cache: compare shares, not absolutes)",
             f"{'kernel':70s} {'launches':>8s} {'ms':>10s} {'share':>7s}"]
    for name in sorted(agg, key=lambda n: -agg[n][1]):
        n, ms = agg[name]
        lines.append(f"{name:70s} {n:8d} {ms:10.2f} {ms / total:7.1%}")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    if sys.argv[1] == "full":
        full(sys.argv[2], sys.argv[3], float(sys.argv[4]) if len(sys.argv) > 4 else None)
    else:
        launch_list(sys.argv[2], sys.argv[3])
