for v in block warp; do
TN_ROWOPS=$v ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"rowstats|softmax_apply" -c 12 --csv --log-file gpurun_out/rowops_$v.csv python tools/eltwise_bench.py --only tile > /dev/null 2>&1
done
