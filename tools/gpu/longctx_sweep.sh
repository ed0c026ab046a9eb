for cap in 5 5.5 6 6.5 7; do
timeout 400 python tools/bench_longctx.py --heads 8 --lag 1 --cap-gib $cap --horizon greedy --steps 3
done
