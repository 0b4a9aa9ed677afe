timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests_full.log 2>&1; tail -n 1 gpurun_out/gpu_tests_full.log
timeout 300 python __graft_entry__.py smoke
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; python -c "import json; d=json.loads(open('gpurun_out/bench.json').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['e2e']['value'], d['roofline']['frac'], d['roofline']['kernel_ms'], d['clocks'])"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:clique_enum -s 1 -c 1 -o gpurun_out/clique_k8 python scripts/prof_clique.py 8 > gpurun_out/ncu_clique.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-extras --cpu-budget 0 > gpurun_out/b_ncu.log 2>&1
