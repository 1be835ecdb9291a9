# full GPU suite + smoke after the fp16 / hp changes and the W8A8 parity restatement
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -rf -s > gpurun_out/suite_tests.log 2>&1; tail -3 gpurun_out/suite_tests.log
grep -E "rows identical|GPU-vs-GPU|^FAILED" gpurun_out/suite_tests.log | cut -c1-300
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
