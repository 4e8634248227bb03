#!/bin/bash
# GPU parity tests on the -DGHN_ASSERTS build (gpurun_alt/libghn_assert.so): shared-memory
# bounds of the thread kernels checked by device asserts.  Restores the product library.
cp paper_2004_02290_b200/libghn.so /tmp/libghn_main.so
cp gpurun_alt/libghn_assert.so paper_2004_02290_b200/libghn.so
python -m pytest tests/test_gpu_thread_kernel.py tests/test_gpu_configs.py tests/test_gpu_edges.py tests/test_gpu_golden.py tests/test_gpu_neighbors.py tests/test_gpu_fullsize.py -q -m gpu 2>&1 | tail -4
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
python tools/robust2d.py 2>&1 | tail -13
cp /tmp/libghn_main.so paper_2004_02290_b200/libghn.so
