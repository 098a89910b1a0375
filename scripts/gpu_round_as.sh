python -c "import __graft_entry__ as g; g.build(); g.smoke(); print('smoke ok')" > gpurun_out/as_smoke.log 2>&1
timeout 2000 python -m pytest tests -m gpu -q > gpurun_out/as_pytest.log 2>&1; echo rc=$? >> gpurun_out/as_pytest.log
timeout 900 python bench.py > gpurun_out/as_bench_default.json 2> gpurun_out/as_bench_default.err
