# ncu full captures of k_pass<32,1,0> (512-row 3-layer) and k_pass<128,1,0> (128-row 2-layer), C4 oneshot
cd $GRAFT_REPO_ROOT
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"k_pass<.int.32, .int.1, .bool.0>" -s 100 -c 1 -o gpurun_out/prof_t32b python bench.py --oneshot --steps 1 --warmup 0 > gpurun_out/prof_t32b.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"k_pass<.int.128, .int.1, .bool.0>" -s 40 -c 1 -o gpurun_out/prof_t128b python bench.py --oneshot --steps 1 --warmup 0 > gpurun_out/prof_t128b.log 2>&1
ls gpurun_out/*.ncu-rep
