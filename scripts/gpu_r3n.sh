# ncu --set full of the final interp kernel at C3e4 (the C4 launch is too long for the full set)
mkdir -p gpurun_out
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"interp_subg" -s 1 -c 1 -o gpurun_out/fin2_full_interp_c3e4 python bench.py --config c3e4 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/fin2_ncu_interp_c3e4.log 2>&1; echo "ncu rc=$?" >> gpurun_out/fin2_ncu_interp_c3e4.log
