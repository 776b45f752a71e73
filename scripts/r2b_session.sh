mkdir -p gpurun_out/r2b
timeout 180 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2b/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r2b/status.txt
if grep -q "smoke ok" gpurun_out/r2b/smoke.log; then
  timeout 1200 python -m pytest tests -m gpu -q -x --timeout 600 > gpurun_out/r2b/tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r2b/status.txt
  timeout 600 python bench.py --no-cpu-baseline > gpurun_out/r2b/bench.json 2> gpurun_out/r2b/bench.err; echo "bench rc=$?" >> gpurun_out/r2b/status.txt
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_leaf_fwd_i8 -s 3 -c 1 -o gpurun_out/r2b/i8 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --small-batch 0 > gpurun_out/r2b/ncu.log 2>&1; echo "ncu rc=$?" >> gpurun_out/r2b/status.txt
fi
