# Round-end evidence on one B200: GPU suite, bench (both arms), launch list, ncu captures.
set -u
O=gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > $O/f_gpu_tests.log 2>&1; echo "tests rc=$?" >> $O/f_gpu_tests.log
python bench.py > $O/f_bench.json 2> $O/f_bench.err
python bench.py --impl reference > $O/f_bench_ref.json 2> $O/f_bench_ref.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/f_launches.csv \
  python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-scenes --no-alt --no-parity-sample > $O/f_launch_run.log 2>&1
python profiles/summarize_launches.py $O/f_launches.csv > $O/f_launches.txt 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_batch_warp -s 8 -c 1 -o /tmp/f_warp \
  python bench.py --steps 3 --warmup 5 --no-alt --no-cpu-baseline --no-scenes --no-parity-sample > $O/f_ncu_warp.log 2>&1
python profiles/summarize_ncu.py /tmp/f_warp.ncu-rep $O/r2f_warp_fp64 --sass --traffic "k_batch_warp<double>" paper_1907_04587_b200/csrc/nsd_k_warp.cu > $O/f_warp_sum.json 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_batch_collide -s 8 -c 1 -o /tmp/f_col \
  python bench.py --steps 3 --warmup 5 --no-alt --no-cpu-baseline --no-scenes --no-parity-sample > $O/f_ncu_col.log 2>&1
python profiles/summarize_ncu.py /tmp/f_col.ncu-rep $O/r2f_collide_fp64 --traffic "k_batch_collide<double>" paper_1907_04587_b200/csrc/nsd_k_warp.cu > $O/f_col_sum.json 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_single_grid -s 3 -c 1 -o /tmp/f_c2 \
  python bench.py --workload c2 --steps 2 --warmup 2 --no-cpu-baseline > $O/f_ncu_c2.log 2>&1
python profiles/summarize_ncu.py /tmp/f_c2.ncu-rep $O/r2f_single_c2_fp64 --sass > $O/f_c2_sum.json 2>&1
cp profiles/dram_traffic.json $O/f_dram_traffic.json
