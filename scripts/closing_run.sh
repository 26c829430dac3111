set -u
O=gpurun_out/${1:-final}
mkdir -p $O
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo rc=$? >> $O/smoke.log
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest.log 2>&1; echo rc=$? >> $O/pytest.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err
for v in 1sm 2sm; do
  timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none -k regex:sk_gemm --csv --log-file $O/skinny_ncu_$v.csv \
    python scripts/skinny_launch.py --variant $v > $O/skinny_launch_$v.json 2>> $O/err.log
done
