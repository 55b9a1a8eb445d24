#!/bin/bash
# L2 atomic / reduction requests of one wt_build per config:
# lts__t_requests_op_{atom,red}.sum summed over the build's kernels, plus
# per-kernel DRAM bytes.  Run on the GPU box; parse with tools/ncu_atomics.py.
set -e
M=lts__t_requests_op_atom.sum,lts__t_requests_op_red.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
for c in ${CFGS:-3 4 5}; do
  python tools/one_build.py $c 0 2 > gpurun_out/atom_plain_$c.log 2>&1
  ncu --metrics $M --clock-control none --csv --log-file gpurun_out/atomics_cfg$c.csv python tools/one_build.py $c 0 2 > gpurun_out/atom_ncu_$c.log 2>&1
done
