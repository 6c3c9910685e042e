cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?"; tail -3 gpurun_out/pytest_gpu.log
ENVS=";FFST_PATH=cta" CFGS="2 3" timeout 600 bash scripts/gpu_env.sh
timeout 300 python bench.py --config 2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c2.json 2>&1; python -c "
import json; d=json.load(open('gpurun_out/bench_c2.json')); print('cufft', d.get('cufft_line'))"
