for v in _ms; do
FDE_LIB=$PWD/paper_1912_13304_b200/libfde${v}.so timeout 600 python tools/sweep.py --only 4 > gpurun_out/sweep4$v.jsonl 2> gpurun_out/sweep4$v.err
python -c "
import json
for l in open('gpurun_out/sweep4$v.jsonl'):
    d = json.loads(l)
    print('$v', d['cfg'], d['n'], 'it/s %.0f' % d['iters_per_s'], 'us/it %.1f' % d['us_per_iter'], {k: round(v/30,1) for k, v in d['loop_body_kernels_us'].items()})
"
done
