mkdir -p gpurun_out
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"bin_|scan_|scatter|spread|interp|pad_|trunc|fft|weights|halo|pif_|migrate" -c 200 --csv --log-file gpurun_out/launches_c4n_r02u.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-pif > gpurun_out/ncu_launch_c4n_r02u.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_launch_c4n_r02u.log
