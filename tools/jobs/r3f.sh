# round 2 (3f): full GPU suite on the cleaned kernel + the headline bench line
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r3f_tests.log 2>&1; echo "tests exit $?" >> gpurun_out/r3f_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r3f_smoke.log 2>&1
python bench.py --steps 20 --warmup 5 > gpurun_out/r3f_bench.json 2> gpurun_out/r3f_bench.err
