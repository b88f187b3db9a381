# ncu full captures of the 512-row T=32 pass and the 128-row T=128 pass (C4 oneshot)
cd $GRAFT_REPO_ROOT
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"k_pass<.int.32, .int.1>" -s 100 -c 1 -o gpurun_out/prof_t32 python bench.py --oneshot --steps 1 --warmup 0 > gpurun_out/prof_t32.log 2>&1
ls gpurun_out/*.ncu-rep
