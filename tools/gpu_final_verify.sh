# Round-end check of the committed tree on one B200: the GPU suite, smoke(),
# the default bench line and the reference arm (the driver's own commands)
O=gpurun_out/fin; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo EXIT $? >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1; echo EXIT $? >> $O/smoke.log
timeout 600 python bench.py > $O/bench.log 2>&1; echo EXIT $? >> $O/bench.log
timeout 600 python bench.py --impl reference > $O/bench_ref.log 2>&1; echo EXIT $? >> $O/bench_ref.log
