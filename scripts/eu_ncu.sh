# euclid evidence: ncu launch list of one 4096x16384 projection + a full capture of the column sort
mkdir -p gpurun_out
TAG=${1:-x}
SHAPES=4096x16384 RELS=0.1 REPS=1 python scripts/time_euclid.py > /dev/null 2>&1
SHAPES=4096x16384 RELS=0.1 REPS=1 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_eu|k_apply|k_colparams" -c 12 --csv --log-file gpurun_out/eu_launches_$TAG.csv python scripts/time_euclid.py > gpurun_out/ncu_eul_$TAG.log 2>&1; echo list=$?
SHAPES=4096x16384 RELS=0.1 REPS=1 ncu --set full --clock-control none -k regex:k_eu_sort -c 1 -o gpurun_out/prof_eu_$TAG -f python scripts/time_euclid.py > gpurun_out/ncu_eu_$TAG.log 2>&1; echo ncu=$?
