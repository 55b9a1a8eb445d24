# per-config report: timing, then one ncu pass per config (DRAM bytes + instructions of every kernel)
mkdir -p gpurun_out; rm -f gpurun_out/report_time.jsonl
timeout 600 python tools/report_time.py 1 2 3 4 5
for c in 1 2 3 4 5; do
  timeout 300 python tools/one_build.py $c 0 1 > /dev/null 2>&1 || exit 1
  timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,sm__inst_executed.sum --clock-control none \
    --csv --log-file gpurun_out/report_ncu_cfg$c.csv python tools/one_build.py $c 0 1 > /dev/null 2>&1
done
ls -la gpurun_out | grep report
