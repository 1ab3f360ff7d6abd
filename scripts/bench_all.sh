# Every bench line of the round into gpurun_out/bench_<tag>.json (one GPU)
set -u
mkdir -p gpurun_out
run() { tag=$1; shift; timeout 900 python bench.py "$@" > gpurun_out/bench_$tag.log 2>&1; grep '^{' gpurun_out/bench_$tag.log | tail -1 > gpurun_out/bench_$tag.json; echo "$tag rc=$?"; }
run C2 --config C2
run C2f32 --config C2f32
run C3 --config C3
run C4 --config C4
run C2_cyclic --config C2 --mode cyclic
run C2_async --config C2 --mode async
run C3_cyclic --config C3 --mode cyclic --steps 10
run C5 --config C5 --steps 3 --warmup 3
run ref_C2 --impl reference --config C2 --steps 2 --warmup 3
