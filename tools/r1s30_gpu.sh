timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r1s30_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r1s30_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r1s30_smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/r1s30_bench.json 2> gpurun_out/r1s30_bench.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r1s30_bench_ref.json 2> gpurun_out/r1s30_bench_ref.err
timeout 1200 python tools/sweep_templates.py > gpurun_out/r1s30_sweep.jsonl 2> gpurun_out/r1s30_sweep.err
