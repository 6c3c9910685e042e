#!/usr/bin/env bash
# One runner for the GPU box (run under gpurun from the repo root; output lands in gpurun_out/).
#   bash scripts/gpu.sh build                         build libffst.so (normally already built here)
#   bash scripts/gpu.sh test [pytest args...]         the -m gpu suite
#   bash scripts/gpu.sh smoke                         __graft_entry__.smoke()
#   bash scripts/gpu.sh bench "<cfgs>" [bench args]   one bench line per config -> gpurun_out/bench_c<C>.json
#   bash scripts/gpu.sh launches <cfg> <tag>          ncu launch list (gpu__time_duration, serialised)
#   bash scripts/gpu.sh prof <cfg> <tag> [kernel-regex] [skip] [count]   ncu --set full capture
#   bash scripts/gpu.sh env "<A=1 B=2;A=2>" "<cfgs>"  bench each ';'-separated environment set
#   bash scripts/gpu.sh traffic <cfg> <tag>           ncu DRAM bytes per launch of the main kernels
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
task=$1; shift
summ() {   # one-line summary of a bench JSON line
  python - "$1" <<'PY'
import json, sys
d = json.load(open(sys.argv[1])); r = d["roofline"]; k = r["kernel_ms"]
print("%s img/s %.1f step %.4f ms | fwd %.4f inv %.4f | %s frac %.3f traffic %s | e2e %s | cpu %s | clocks %s" % (
    d["config"]["workload"], d["value"], d["ms_per_step"], k["fwd_main"], k["inv_main"], r["kernel"], r["frac"],
    r.get("traffic"), (d.get("e2e") or {}).get("value"), (d.get("cpu_baseline") or {}).get("value"),
    (d.get("clocks") or {}).get("sm_mhz")))
PY
}
case "$task" in
  build) python -c "import __graft_entry__ as g; g.build()" ;;
  test) timeout 2400 python -m pytest tests -q -m gpu "$@" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?"
        tail -5 gpurun_out/pytest_gpu.log ;;
  smoke) timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2 ;;
  bench) cfgs=$1; shift
    for c in $cfgs; do
      timeout 1200 python bench.py --config "$c" "$@" > gpurun_out/bench_c$c.json 2> gpurun_out/bench_c$c.err
      echo "bench c$c exit $?"; summ gpurun_out/bench_c$c.json || tail -3 gpurun_out/bench_c$c.err
    done ;;
  launches) c=$1; tag=$2
    CMD="python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline --no-cufft"
    timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
      --log-file gpurun_out/launches_$tag.csv $CMD > gpurun_out/launches_$tag.log 2>&1; echo "ncu launches exit $?" ;;
  prof) c=$1; tag=$2; kr=${3:-main_kernel}; s=${4:-2}; cnt=${5:-2}
    CMD="python bench.py --config $c --steps 1 --warmup 1 --no-cpu-baseline --no-cufft"
    $CMD > gpurun_out/plain_$tag.log 2>&1 && timeout 1800 ncu -f --set full --clock-control none --import-source on \
      -k regex:$kr -s $s -c $cnt -o /tmp/prof_$tag $CMD > /tmp/ncu_$tag.log 2>&1; echo "ncu exit $?"
    tail -2 /tmp/ncu_$tag.log
    ncu -i /tmp/prof_$tag.ncu-rep --page raw --csv > gpurun_out/prof_${tag}_raw.csv 2>&1
    ncu -i /tmp/prof_$tag.ncu-rep --page details --csv > gpurun_out/prof_${tag}_details.csv 2>&1
    ncu -i /tmp/prof_$tag.ncu-rep --page source --csv --print-source cuda,sass > /tmp/src.csv 2>&1
    gzip -c /tmp/src.csv > gpurun_out/prof_${tag}_source.csv.gz ;;
  traffic) c=$1; tag=$2   # DRAM bytes per launch of the two persistent kernels (one eager step after warm-up)
    CMD="python bench.py --config $c --steps 1 --warmup 1 --no-cpu-baseline --no-cufft --no-graph"
    timeout 1800 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
      -k regex:"main_kernel|tiny_" --csv --log-file gpurun_out/traffic_$tag.csv $CMD > gpurun_out/traffic_$tag.log 2>&1
    echo "ncu traffic exit $?" ;;
  env) IFS=';' read -ra SETS <<< "$1"; cfgs=$2
    for e in "${SETS[@]}"; do for c in $cfgs; do
      env $e timeout 600 python bench.py --config "$c" --steps ${STEPS:-5} --warmup 3 --no-cpu-baseline --no-cufft \
        > gpurun_out/b.json 2> gpurun_out/b.err || tail -2 gpurun_out/b.err
      echo -n "[$e] "; summ gpurun_out/b.json
    done; done ;;
  *) echo "unknown task $task"; exit 2 ;;
esac
