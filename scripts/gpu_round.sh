# round-end style refresh: bench (both arms), launch list, clique + motif ncu, shard balance, extras
set -x
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -n 1 gpurun_out/bench.json | cut -c1-300
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-extras --cpu-budget 0 > gpurun_out/b_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:clique_enum -s 1 -c 1 -o gpurun_out/clique_k8 python scripts/prof_clique.py 8 > gpurun_out/ncu_clique.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:motif_enum -s 1 -c 1 -o gpurun_out/motif_cfg4_k5 python scripts/prof_motif.py cfg4 5 16384 > gpurun_out/ncu_motif.log 2>&1
timeout 900 python scripts/shard_scaling.py > gpurun_out/shard_scaling.jsonl 2> gpurun_out/shard_scaling.err
timeout 1500 python scripts/bench_extras.py --full > gpurun_out/extras.jsonl 2> gpurun_out/extras.err; tail -n 3 gpurun_out/extras.err
echo done
