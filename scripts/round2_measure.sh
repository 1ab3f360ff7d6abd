# Round-2 evidence on one GPU: every bench line, the reference arm, the
# persistent-sweep trace, launch lists and ncu --set full captures of the
# dense correlation (H) at C2 fp64 / C2 fp32 / C3 fp32.  Outputs: gpurun_out/r2/
set -u
O=gpurun_out/r2
mkdir -p $O
run() { tag=$1; shift; timeout 900 python bench.py "$@" > $O/bench_$tag.log 2>&1; grep '^{' $O/bench_$tag.log | tail -1 > $O/bench_$tag.json; echo "$tag rc=$?"; }
( time run C2 --config C2 ) 2>&1 | tail -4
run C2f32 --config C2f32
run C3 --config C3
run C4 --config C4
run C2_cyclic --config C2 --mode cyclic
run C2_async --config C2 --mode async
run C5 --config C5 --steps 3 --warmup 3
run ref_C2 --impl reference --config C2 --steps 5 --warmup 2
BD3MG_PK=1 timeout 300 python scripts/pk_trace.py C2 > $O/pk_trace_C2.txt 2>&1
python scripts/sweep_timeline.py C2 3 > $O/timeline_C2.md 2>/dev/null
python scripts/prof_sweep_cfg.py C2 2 > /dev/null
ncu --metrics gpu__time_duration.sum,sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active,dram__bytes.sum \
    --clock-control none --csv --log-file $O/sweep_kernels_C2.csv python scripts/prof_sweep_cfg.py C2 2 > /dev/null 2>&1
python scripts/launch_metrics.py $O/sweep_kernels_C2.csv 14 > $O/sweep_kernels_C2.md
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_sweep_C2.csv \
    python scripts/prof_sweep_cfg.py C2 3 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_bench.csv \
    python bench.py --steps 3 --warmup 3 --quick > /dev/null 2>&1
for c in C2 C2f32 C3; do
  python scripts/prof_h_cfg.py $c 2 > /dev/null
  ncu --set full --clock-control none --import-source on -k regex:conv_ -c 1 -o $O/H_$c \
      python scripts/prof_h_cfg.py $c 1 > /dev/null 2>&1
done
ls -la $O
python -m pytest tests -q -m gpu > $O/gpu_tests.txt 2>&1; tail -3 $O/gpu_tests.txt
python __graft_entry__.py --smoke >> $O/gpu_tests.txt 2>&1; tail -1 $O/gpu_tests.txt
