cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.max.sm,memory.total --format=csv,noheader
timeout 900 python bench.py > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; tail -c 400 gpurun_out/bench_c4.json; echo
timeout 300 python bench.py --config c2 > gpurun_out/bench_c2.json 2>&1; tail -c 200 gpurun_out/bench_c2.json; echo
timeout 300 python bench.py --config c3 --no-cpu-baseline > gpurun_out/bench_c3.json 2>&1; tail -c 200 gpurun_out/bench_c3.json; echo
timeout 300 python bench.py --config c1 > gpurun_out/bench_c1.json 2>&1; tail -c 200 gpurun_out/bench_c1.json; echo
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_c4.json 2>&1; tail -c 300 gpurun_out/bench_ref_c4.json; echo
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4_v3.csv python bench.py --oneshot --steps 1 --warmup 0 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_layer_bulk -s 300 -c 1 -o gpurun_out/prof_c4_v3 python bench.py --oneshot --steps 1 --warmup 0 > gpurun_out/prof_c4_v3.log 2>&1; tail -1 gpurun_out/prof_c4_v3.log
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -k full_size_c4 2>&1 | tail -2
