"""Summarises an .ncu-rep (read here, without a GPU) into the few numbers the
roofline discussion needs. Usage: python tools/ncu_summary.py rep [rep ...]"""
import csv
import io
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__warps_active.avg.per_cycle_active",
    "smsp__warps_eligible.avg.per_cycle_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_issued.avg.pct_of_peak_sustained_active",
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def main():
    for rep in sys.argv[1:]:
        hdr, units, rows = raw(rep)
        idx = {h: i for i, h in enumerate(hdr)}
        for r in rows:
            print("=" * 100)
            print(rep, "|", r[idx["Kernel Name"]][:90])
            for k in KEYS:
                if k in idx:
                    print(f"  {k:75s} {r[idx[k]]:>18s} {units[idx[k]]}")
            st = [(h, float(r[i])) for h, i in idx.items()
                  if h.startswith("smsp__average_warps_issue_stalled") and h.endswith("per_issue_active.ratio")]
            print("  stalls per issue:", ", ".join(f"{h[34:-23]}={v:.2f}" for h, v in sorted(st, key=lambda x: -x[1])[:7]))
            d = {k: float(r[idx[k]].replace(",", "")) for k in KEYS if k in idx and r[idx[k]] not in ("", "n/a")}
            t = d.get("gpu__time_duration.sum")
            unit = units[idx["gpu__time_duration.sum"]]
            sec = t * {"ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1.0, "usecond": 1e-6, "msecond": 1e-3, "nsecond": 1e-9}.get(unit, 1e-9)
            def per_cycle(op):
                k = f"smsp__sass_thread_inst_executed_op_{op}_pred_on.sum.per_cycle_elapsed"
                return float(r[idx[k]].replace(",", "")) if k in idx and r[idx[k]] not in ("", "n/a") else 0.0
            cyc = float(r[idx["sm__cycles_elapsed.avg"]].replace(",", "")) if "sm__cycles_elapsed.avg" in idx else 0.0
            dp = (per_cycle("dfma"), per_cycle("dmul"), per_cycle("dadd"))
            sp = (per_cycle("ffma"), per_cycle("fmul"), per_cycle("fadd"))
            f64 = (2 * dp[0] + dp[1] + dp[2]) * cyc
            f32 = (2 * sp[0] + sp[1] + sp[2]) * cyc
            print(f"  FP64 thread-instr/cycle (chip): dfma {dp[0]:.0f} dmul {dp[1]:.0f} dadd {dp[2]:.0f} "
                  f"= {sum(dp):.0f} of 9472 issue slots ({sum(dp) / 9472:.1%})")
            if sum(sp) > 0:
                print(f"  FP32 thread-instr/cycle (chip): ffma {sp[0]:.0f} fmul {sp[1]:.0f} fadd {sp[2]:.0f} "
                      f"= {sum(sp):.0f} of 18944 issue slots ({sum(sp) / 18944:.1%})")
            print(f"  hardware-counted FLOP/s: fp64 {f64 / sec / 1e12:.2f} TF, fp32 {f32 / sec / 1e12:.2f} TF  "
                  f"(duration {sec * 1e3:.4f} ms, {cyc:.0f} SM cycles)")


if __name__ == "__main__":
    main()
