for d in 0 1 2 3; do EINET_CT_DEBUG=$d timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/ctexp/b$d.json 2>/dev/null; done
