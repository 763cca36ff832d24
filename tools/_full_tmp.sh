mkdir -p gpurun_out/full
timeout 2000 python -m pytest tests -m gpu -q -x -p no:cacheprovider --durations=15 > gpurun_out/full/pytest.log 2>&1; echo "pytest rc=$?"
tail -25 gpurun_out/full/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -3
timeout 900 python bench.py > gpurun_out/full/bench.json 2> gpurun_out/full/bench.err; echo "bench rc=$?"; tail -c 3000 gpurun_out/full/bench.json
