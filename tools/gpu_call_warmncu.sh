#!/bin/bash
# Warm-cache (no flush between kernels) DRAM/L2 counters of the sine-domain
# PCG iteration kernels: one pass per kernel (no replay), --cache-control none.
mkdir -p gpurun_out
FDE_GRAPH=0 timeout 600 ncu --cache-control none --clock-control none \
  --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_write.sum \
  -k regex:"k_sop|k_sine_xr5" -s 20 -c 6 --csv python tools/unit_run.py --reps 1 --pcg > gpurun_out/warmncu.csv 2> gpurun_out/warmncu.err
echo "ncu rc=$?"
python - <<'PY'
import csv
rows=[r for r in csv.reader(open('gpurun_out/warmncu.csv')) if len(r)>10]
h=rows[0]
ik=h.index('Kernel Name'); im=h.index('Metric Name'); iv=h.index('Metric Value'); iid=h.index('ID')
for r in rows[1:]:
    print(r[iid], r[ik][:22], r[im], r[iv])
PY
