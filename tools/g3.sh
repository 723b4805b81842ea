# ncu evidence for the bench line (launch list of the same command + one --set full capture of the top kernels)
export CUDA_DEVICE_MAX_CONNECTIONS=32
O=gpurun_out/${TAG:-r02c}; WL=${WL:-C2}; mkdir -p $O
timeout 600 python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_$WL.csv \
  python bench.py --workload $WL --steps 1 --warmup 1 --no-cpu-baseline > $O/launches_$WL.log 2>&1
echo "ncu launches exit $?" >> $O/launches_$WL.log
timeout 1200 ncu --set full --clock-control none --import-source on -k "regex:gemm|merge|attention|norm" -s 60 -c 14 \
  -o $O/full_$WL python bench.py --workload $WL --steps 1 --warmup 1 --no-cpu-baseline > $O/full_$WL.log 2>&1
echo "ncu full exit $?" >> $O/full_$WL.log
ls -la $O
