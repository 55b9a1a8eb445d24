# per-kernel launch list of hwt_build (second build of each input)
mkdir -p gpurun_out
for w in cfg4 zipf2.0 cfg3; do
  timeout 300 python tools/hwt_one.py $w || exit 1
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/hwt_launches_$w.csv python tools/hwt_one.py $w > /dev/null 2>&1
done
ls -la gpurun_out
