mkdir -p gpurun_out/wsexp
for d in 0 1 2 3; do EINET_WS_DEBUG=$d timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/wsexp/b$d.json 2>/dev/null; done
