mkdir -p gpurun_out
timeout 300 python tools/ab_sop.py 2>&1 | sed "s/^/[persist] /"
FDE_GRAPH=body timeout 300 python tools/ab_sop.py 2>&1 | sed "s/^/[body] /"
timeout 900 python -m pytest tests -m gpu -x -q -k "pcg or sine or solver_parity or parity_full" 2>&1 | tail -5
