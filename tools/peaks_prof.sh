# Fine-grained ncu stall sampling of the peak kernels on cfg2 / cfg5
# (single frames: latency-bound kernels, so the sampling interval is minimal)
set -u
out=gpurun_out; mkdir -p $out
tag=${1:-r02n}
timeout 300 python bench.py --workload cfg2 --profile --steps 2 --warmup 3 > $out/${tag}_cfg2.log 2>&1; echo run=$?
timeout 300 ncu --set full --import-source on --warp-sampling-interval 0 --kernel-name-base demangled -k regex:"peaks_" -s 12 -c 6 -o $out/${tag}_cfg2_peaks -f python bench.py --workload cfg2 --profile --steps 3 --warmup 3 > $out/${tag}_ncu2.log 2>&1; echo ncu2=$?
timeout 300 ncu --set full --import-source on --warp-sampling-interval 0 --kernel-name-base demangled -k regex:"peaks_" -s 12 -c 6 -o $out/${tag}_cfg5_peaks -f python bench.py --workload cfg5 --profile --steps 3 --warmup 3 > $out/${tag}_ncu5.log 2>&1; echo ncu5=$?
