cd $GRAFT_REPO_ROOT
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"k_pass<.int.128, .int.1, .bool.0>" -s 40 -c 1 -o gpurun_out/v13_prof_p128 python bench.py --oneshot --steps 1 --warmup 0 > /dev/null 2>&1
ls gpurun_out/v13_prof_p128.ncu-rep
