python -c "import __graft_entry__ as g; g.build(); g.smoke(); print('smoke ok')" > gpurun_out/ak_smoke.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/ak_pytest.log 2>&1; echo rc=$? >> gpurun_out/ak_pytest.log
timeout 900 python bench.py > gpurun_out/ak_bench_default.json 2> gpurun_out/ak_bench_default.err
timeout 900 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/ak_bench_ref.json 2> gpurun_out/ak_bench_ref.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29871 bench.py --gpus 2 > gpurun_out/ak_bench_n2.json 2> gpurun_out/ak_bench_n2.err
