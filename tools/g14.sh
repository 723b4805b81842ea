export CUDA_DEVICE_MAX_CONNECTIONS=32
TAG=r02n WL=C2 bash tools/gpu_round.sh build smoke suite bench > /dev/null 2>&1
O=gpurun_out/r02n
timeout 900 python bench.py --workload C2p > $O/bench_C2p.json 2> $O/bench_C2p.err
timeout 900 python bench.py --workload C3 --no-cpu-baseline > $O/bench_C3.json 2> $O/bench_C3.err
ls -la $O
