timeout 900 python bench.py > gpurun_out/bench.jsonl 2> gpurun_out/bench.err; echo "bench rc=$?"
tail -3 gpurun_out/bench.err
cat gpurun_out/bench.jsonl
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
