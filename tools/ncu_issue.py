"""Instruction-issue and fp64 counters per launch from `ncu --set full` captures, for the bench
line's `roofline.issue` object (bench.py::_issue).  The kernels are not HBM-bound (k_step: fp64
dependency chains; k_render: fragment instruction issue), so next to the HBM fraction the bench
reports how much of the SMs' instruction-issue capacity a launch uses:

    issue frac = warp instructions per launch / (4 SMSPs x SMs x SM clock x launch time)

with the warp-instruction count from ncu (it does not change with the clock) and the launch time
measured live.  Usage:

    python tools/ncu_issue.py c2=gpurun_out/X_prof_step.ncu-rep:4096 c3=gpurun_out/X_prof_render.ncu-rep:1024

writes profiles/issue.json (per workload: per-kernel counts and the units of the capture).
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], check=True, capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    units = dict(zip(rows[0], rows[1]))
    return [dict(zip(rows[0], r)) for r in rows[2:]], units


def main():
    path = os.path.join(ROOT, "profiles", "issue.json")
    doc = json.load(open(path)) if os.path.exists(path) else {}
    doc["_doc"] = __doc__.split("\n\n")[0].replace("\n", " ")
    for arg in sys.argv[1:]:
        wl, spec = arg.split("=", 1)
        rep, units = spec.rsplit(":", 1)
        recs, unit = raw(rep)
        to_us = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3, "s": 1e6, "second": 1e6}[unit["gpu__time_duration.sum"]]
        for r in recs:
            name = r["Kernel Name"].split("(")[0].split("<")[0].replace("void ", "").strip()
            cyc = float(r["smsp__cycles_elapsed.avg"])
            f = lambda k: float(r[k].replace(",", "")) * cyc  # noqa: E731 (per-cycle sums -> per launch)
            doc.setdefault(wl, {})[name] = {
                "units": int(units),
                "warp_inst": int(float(r["smsp__inst_executed.sum"].replace(",", ""))),
                "fp64_dfma_thread_ops": int(f("smsp__sass_thread_inst_executed_op_dfma_pred_on.sum.per_cycle_elapsed")),
                "fp64_dadd_thread_ops": int(f("smsp__sass_thread_inst_executed_op_dadd_pred_on.sum.per_cycle_elapsed")),
                "fp64_dmul_thread_ops": int(f("smsp__sass_thread_inst_executed_op_dmul_pred_on.sum.per_cycle_elapsed")),
                "ncu_issue_active": float(r["smsp__issue_active.avg.pct_of_peak_sustained_active"]) / 100,
                "ncu_fp64_pipe_active": float(r["sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"]) / 100,
                "ncu_us": float(r["gpu__time_duration.sum"].replace(",", "")) * to_us,
                "_capture": os.path.basename(rep) + " (tools/gpu_round.sh)",
            }
    with open(path, "w") as fh:
        json.dump(doc, fh, indent=1)
    print(json.dumps(doc, indent=1))


if __name__ == "__main__":
    main()
