#!/bin/bash
# Copy / summarise one tools/gpu_round.sh (+ tools/env_sweep.sh) run into profiles/ (here, no GPU):
#   bash tools/refresh_profiles.sh TAG      (reads gpurun_out/TAG_*)
set -e
T=${1:?tag}; G=gpurun_out; P=profiles
python tools/ncu_summary.py rep $G/${T}_prof_step.ncu-rep > $P/r02_k_step_ncu.csv
python tools/ncu_summary.py rep $G/${T}_prof_render.ncu-rep > $P/r02_k_render_ncu.csv
python tools/ncu_summary.py launches $G/${T}_launches.csv > $P/r02_launches_summary.csv
python tools/ncu_lines.py $G/${T}_prof_step.ncu-rep paper_2410_00425_b200/_lib/step.o k_step 40 > $P/r02_k_step_lines.txt 2>&1
python tools/ncu_lines.py $G/${T}_prof_render.ncu-rep paper_2410_00425_b200/_lib/raster.o k_render 40 raster.cu:800-850 > $P/r02_k_render_lines.txt 2>&1
cp $G/${T}_phase.txt $P/r02_k_step_phases.txt
(echo "# racecheck / memcheck (tools/sanitize.sh, $T): small probes of every task + rasterizer, and the benchmark-scale probe (>= 3 frames per persistent rasterizer CTA, a full 4096-env step wave)"
 for f in racecheck racecheck_scale memcheck memcheck_scale; do echo "## $f"; cat $G/${T}_$f.txt; done) > $P/r02_sanitizer.txt
for f in bench bench_ref bench_ref_c3 bench_ref_c4 bench_ref_c5 bench_c4 bench_c5 bench_2rank; do cp $G/${T}_$f.json $P/r02_$f.json; done
[ -f $G/${T}_sweep_c2.jsonl ] && cp $G/${T}_sweep_c2.jsonl $P/r02_c2_env_sweep.jsonl
[ -f $G/${T}_sweep_c3.jsonl ] && cp $G/${T}_sweep_c3.jsonl $P/r02_c3_env_sweep.jsonl
rm -f $P/issue.json
python tools/ncu_issue.py c2=$G/${T}_prof_step.ncu-rep:4096 c3=$G/${T}_prof_render.ncu-rep:1024 \
  c4=$G/${T}_issue_render_c4.ncu-rep:1024 c5=$G/${T}_issue_render_c5.ncu-rep:1024 > /dev/null
python - "$T" <<'PY'
import csv, io, json, subprocess, sys
T = sys.argv[1]
t = json.load(open("profiles/traffic.json"))
def dram(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics",
                          "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    d, u = dict(zip(rows[0], rows[2])), dict(zip(rows[0], rows[1]))
    mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    b = sum(float(d[k].replace(",", "")) * mult[u[k]] for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
    return int(b), d["gpu__time_duration.sum"] + " " + u["gpu__time_duration.sum"]
b, tm = dram(f"gpurun_out/{T}_prof_step.ncu-rep")
t["c2"] = {"k_step": b, "_capture": f"{T}_prof_step: 4096 envs, {tm} (profiles/r02_k_step_ncu.csv)"}
b, tm = dram(f"gpurun_out/{T}_prof_render.ncu-rep")
t["c3"] = {"k_render": b, "_capture": f"{T}_prof_render: 1024 envs x 128x128, {tm} (profiles/r02_k_render_ncu.csv)"}
json.dump(t, open("profiles/traffic.json", "w"), indent=1)
PY
echo "profiles refreshed from $T"
