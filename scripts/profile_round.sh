# Round profiles (one GPU): launch lists of the C2 fp64 and C3 fp32 sweeps, and
# full captures of the H kernels (dram traffic per launch for bench.py).
set -u
mkdir -p gpurun_out/prof
python scripts/prof_sweep_cfg.py C2 2 > /dev/null
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/prof/launches_C2.csv \
    python scripts/prof_sweep_cfg.py C2 3 > /dev/null 2>&1
python scripts/prof_sweep_cfg.py C3 2 > /dev/null
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/prof/launches_C3.csv \
    python scripts/prof_sweep_cfg.py C3 2 > /dev/null 2>&1
for c in C2 C2f32 C3; do
  python scripts/prof_h_cfg.py $c 2 > /dev/null
  ncu --set full --clock-control none --import-source on -k regex:conv_ -c 1 -o gpurun_out/prof/H_$c \
      python scripts/prof_h_cfg.py $c 1 > /dev/null 2>&1
done
ls -la gpurun_out/prof
