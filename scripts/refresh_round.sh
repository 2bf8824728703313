# Round evidence refresh: all-config device table (+ reference CPU) and the headline bench line.
mkdir -p gpurun_out
TAG=${1:-x}
timeout 1200 python scripts/bench_configs.py > gpurun_out/configs_$TAG.json 2> gpurun_out/configs_$TAG.err; echo configs=$?
timeout 900 python bench.py > gpurun_out/bench_$TAG.log 2>&1; echo bench=$?
