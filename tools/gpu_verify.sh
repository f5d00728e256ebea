cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/v1
nvidia-smi --query-gpu=name,clocks.max.sm,memory.total --format=csv > gpurun_out/v1/smi.txt
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/v1/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/v1/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/v1/smoke.log 2>&1
python bench.py > gpurun_out/v1/bench.json 2> gpurun_out/v1/bench.err
python bench.py --case ensemble > gpurun_out/v1/bench_ens.json 2>/dev/null
tail -3 gpurun_out/v1/pytest_gpu.log; cat gpurun_out/v1/bench.json | head -c 600
