# K19 build-variant sweep: bash tools/exp/epi.sh "<NVEXTRA flags>" ...
mkdir -p gpurun_out
for X in "$@"; do
  make -C paper_1904_09538_b200/csrc clean >/dev/null 2>&1
  make -C paper_1904_09538_b200/csrc -j16 NVEXTRA="$X" >/dev/null 2>&1 || echo build-fail
  echo "== $X" >> gpurun_out/epi.log
  timeout 300 python -m pytest -q -x tests/test_gpu_dg_tc.py 2>&1 | tail -1 >> gpurun_out/epi.log
  timeout 300 python tools/exp/dg_tc_time.py 2>&1 | cut -c1-60 >> gpurun_out/epi.log
done
