A="--heads 8 --lag 1 --cap-gib 6 --horizon greedy --steps 4"
timeout 300 python tools/bench_longctx.py $A
timeout 300 python tools/bench_longctx.py $A --pv-ksplit 4
timeout 300 python tools/bench_longctx.py $A
timeout 300 python tools/bench_longctx.py $A --pv-ksplit 4
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"gemm" -c 60 --csv --log-file gpurun_out/lc_gemm_ks.csv python tools/bench_longctx.py --heads 8 --lag 1 --cap-gib 6 --horizon greedy --steps 1 --pv-ksplit 4 > /dev/null 2>&1
