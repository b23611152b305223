mkdir -p gpurun_out/final
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final/smoke.txt 2>&1; echo smoke=$?
timeout 2400 python -m pytest tests -m gpu -q 2>&1 | tail -3 > gpurun_out/final/gpu_tests.txt
timeout 900 python bench.py > gpurun_out/final/bench.json 2> gpurun_out/final/bench.err; echo bench=$?
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/final/bench_ref.json 2>> gpurun_out/final/bench.err; echo ref=$?
cat gpurun_out/final/gpu_tests.txt
