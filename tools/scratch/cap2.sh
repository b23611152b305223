bash tools/capture_r02.sh
timeout 900 python bench.py > gpurun_out/r02/bench.json 2> gpurun_out/r02/bench.err; echo bench=$?
