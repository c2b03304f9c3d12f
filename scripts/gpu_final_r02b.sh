#!/bin/bash
# round-2 final evidence (after the setpts L2 hints): smoke, GPU suite, default bench
# line (C4), reference arm, the ncu launch list of the same command, one --set full
# capture of the spread kernel and a dram-only capture of the interp kernel (the full
# set times out on the 190 ms interp launch and reports nan)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fin2_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/fin2_smoke.log
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/fin2_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/fin2_tests.log
timeout 900 python bench.py > gpurun_out/fin2_bench.json 2> gpurun_out/fin2_bench.err; echo "bench rc=$?" >> gpurun_out/fin2_bench.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/fin2_ref.json 2> gpurun_out/fin2_ref.err
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"bin_|scan_|scatter|spread|interp|pad_|trunc|fft|weights|halo|pif_|migrate" -c 300 --csv --log-file gpurun_out/fin2_launches_c4n.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-pif > gpurun_out/fin2_ncu_launch.log 2>&1; echo "ncu launch rc=$?" >> gpurun_out/fin2_ncu_launch.log
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"spread_subg" -s 1 -c 1 -o gpurun_out/fin2_full_spread python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-pif > gpurun_out/fin2_ncu_full.log 2>&1; echo "ncu full rc=$?" >> gpurun_out/fin2_ncu_full.log
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,smsp__inst_executed.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,lts__t_sector_hit_rate.pct --clock-control none -k regex:"interp_subg" -s 1 -c 1 -o gpurun_out/fin2_dram_interp python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-pif > gpurun_out/fin2_ncu_interp.log 2>&1; echo "ncu interp rc=$?" >> gpurun_out/fin2_ncu_interp.log
