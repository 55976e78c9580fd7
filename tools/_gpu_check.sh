# quick GPU iteration: parity tests, smoke, bench, per-config rates
tag=${1:-x}
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${tag}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${tag}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${tag}_smoke.log 2>&1
timeout 400 python bench.py > gpurun_out/${tag}_bench.log 2>&1
timeout 300 python tools/bench_configs.py > gpurun_out/${tag}_configs.log 2>&1
