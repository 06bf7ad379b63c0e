"""Summarise an ncu --set full capture of the engine kernel into profiles/.

    python scripts/ncu_summary.py gpurun_out/prof.ncu-rep --trials 209715200 \
        --out profiles/r01_v2_f32_ncu

writes <out>.json (the numbers bench.py reads: DRAM bytes per trial, issue
activity) and <out>.md (pipes, stalls, instruction mix per trial, hottest
SASS lines).  Runs here, without a GPU (ncu -i).
"""
import argparse
import collections
import csv
import json
import subprocess


def raw_metrics(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, units, v = rows[0], rows[1], rows[2]
    return {k: (v[i], units[i]) for i, k in enumerate(h)}


def sass_rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    return rows[0], rows[1], rows[2:]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--trials", type=float, required=True, help="Metropolis trials in the profiled launch")
    ap.add_argument("--out", required=True)
    ap.add_argument("--label", default="")
    a = ap.parse_args()
    m = raw_metrics(a.rep)

    def f(k):
        return float(m[k][0].replace(",", "")) if k in m else float("nan")

    dur_ms = f("gpu__time_duration.sum")
    unit = m.get("gpu__time_duration.sum", ("", ""))[1]
    if unit == "us":
        dur_ms /= 1e3
    elif unit == "ns":
        dur_ms /= 1e6

    def to_bytes(k):
        val, u = m.get(k, ("nan", "byte"))
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
        return float(val.replace(",", "")) * scale

    dram = to_bytes("dram__bytes_read.sum") + to_bytes("dram__bytes_write.sum")
    kname, hdr, data = sass_rows(a.rep)
    ia = hdr.index("Instructions Executed")
    isrc = hdr.index("Source")
    iw = hdr.index("Warp Stall Sampling (All Samples)")
    warp_trials = a.trials / 32
    ops = collections.Counter()
    st = collections.Counter()
    for r in data:
        n = int(r[ia] or 0)
        s = r[isrc].split()
        if not s:
            continue
        op = s[1] if s[0].startswith("@") else s[0]
        ops[op] += n / warp_trials
        st[op] += int(r[iw] or 0)
    tot_st = max(1, sum(st.values()))
    stalls = {k.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""): f(k)
              for k in m if k.startswith("smsp__average_warps_issue_stalled") and k.endswith("per_issue_active.ratio")}
    summary = {
        "label": a.label, "report": a.rep, "kernel": kname[1] if len(kname) > 1 else "",
        "duration_ms": dur_ms, "trials": a.trials, "trials_per_s": a.trials / (dur_ms / 1e3),
        "dram_bytes": dram, "dram_bytes_per_trial": dram / a.trials,
        "issue_active_frac": f("smsp__issue_active.avg.pct_of_peak_sustained_active") / 100,
        "smem_wavefronts": f("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"),
        "smem_bank_conflicts": f("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"),
        "registers_per_thread": f("launch__registers_per_thread"),
        "warps_active_per_sm": f("sm__warps_active.avg.per_cycle_active"),
        "pipe_fma_pct": f("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"),
        "pipe_alu_pct": f("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active"),
        "pipe_fp64_pct": f("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
        "pipe_fmaheavy_pct": f("sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed"),
        "pipe_xu_pct": f("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active"),
        "pipe_lsu_pct": f("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active"),
        "instructions_per_warp_trial": sum(ops.values()),
        "stalls_per_issue": {k: v for k, v in sorted(stalls.items(), key=lambda x: -x[1]) if v > 0.05},
        "instruction_mix_per_warp_trial": {k: round(v, 2) for k, v in ops.most_common(25)},
    }
    with open(a.out + ".json", "w") as fh:
        json.dump(summary, fh, indent=1)
    hot = sorted(data, key=lambda r: -int(r[iw] or 0))[:25]
    with open(a.out + ".md", "w") as fh:
        fh.write(f"# ncu summary: {a.label}\n\n")
        fh.write(f"Kernel: `{summary['kernel']}`  \nReport: `{a.rep}` (ncu --set full --clock-control none)\n\n")
        fh.write("| metric | value |\n|---|---|\n")
        for k in ("duration_ms", "trials", "trials_per_s", "dram_bytes", "dram_bytes_per_trial", "issue_active_frac",
                  "smem_wavefronts", "smem_bank_conflicts", "registers_per_thread", "warps_active_per_sm",
                  "pipe_fma_pct", "pipe_fmaheavy_pct", "pipe_alu_pct", "pipe_fp64_pct", "pipe_xu_pct", "pipe_lsu_pct",
                  "instructions_per_warp_trial"):
            fh.write(f"| {k} | {summary[k]:.6g} |\n")
        fh.write("\n## Stall reasons (warps stalled per issued instruction)\n\n")
        for k, v in summary["stalls_per_issue"].items():
            fh.write(f"- {k}: {v:.2f}\n")
        fh.write("\n## Instruction mix (warp instructions per warp-trial)\n\n")
        for k, v in summary["instruction_mix_per_warp_trial"].items():
            fh.write(f"- {k}: {v} (stall samples {100 * st[k] / tot_st:.1f}%)\n")
        fh.write("\n## Hottest SASS lines (stall samples)\n\n```\n")
        for r in hot:
            fh.write(f"{100 * int(r[iw] or 0) / tot_st:5.1f}%  {int(r[ia] or 0) / warp_trials:6.2f}/trial  {r[isrc][:90]}\n")
        fh.write("```\n")
    print(json.dumps({k: summary[k] for k in ("duration_ms", "trials_per_s", "dram_bytes_per_trial",
                                              "issue_active_frac", "instructions_per_warp_trial")}))


if __name__ == "__main__":
    main()
