#!/bin/bash
# The GPU suite under the device-bounds-checked library (LSV_DEVICE_CHECKS=1), plus the sanitize
# cases: the compute-sanitizer substitute (the tool is closed on the pool).
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_checked.log 2>&1
LSV_EXPECT_CHECKED=1 LSV_LIB_PATH=paper_2511_22880_b200/liblsv_checked.so timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_checked.log 2>&1
echo "checked suite rc=$?"; tail -3 gpurun_out/pytest_checked.log
LSV_LIB_PATH=paper_2511_22880_b200/liblsv_checked.so timeout 900 python tools/sanitize_cases.py > gpurun_out/sanitize_checked.log 2>&1
echo "checked sanitize cases rc=$?"; tail -7 gpurun_out/sanitize_checked.log
