# euclid iteration: GPU tests + timing, radix vs bitonic column sort
mkdir -p gpurun_out
TAG=${1:-x}
timeout 900 python -m pytest tests/test_gpu_euclid.py -x -q > gpurun_out/pytest_eu_$TAG.log 2>&1; echo eu_tests=$?
{ python scripts/time_euclid.py; MP_EU_SORT=bitonic python scripts/time_euclid.py; } > gpurun_out/eu_time_$TAG.log 2>&1; echo time=$?
