#!/bin/bash
# One `ncu --set full` capture per listed suite kernel (inputs resident,
# 1 launch profiled), reports under gpurun_out/ncu_<tag>.ncu-rep, plus the
# launch list of a short bench run. Run on the GPU box via gpurun.
set -u
out=gpurun_out
only=${1:-}
mkdir -p $out
cap() {  # tag kernel-regex variant-id
  if [ -n "$only" ] && [ "$only" != "$1" ] && [ "$only" != "launches" ]; then return; fi
  if [ "$only" = "launches" ]; then return; fi
  timeout 600 ncu --set full --clock-control none --import-source on -k "regex:$2" -s 1 -c 1 \
    -o $out/ncu_$1 -f python tools/run_kernel.py "$3" 2 > $out/ncu_$1.log 2>&1
  echo "$1 rc=$?"
}
cap mm_nopf_8192 matmul_nopf "matmul_sq__dtype-float32__groups_fit-True__lsize_0-16__lsize_1-16__n-8192__prefetch-False"
cap mm_pf_4096 matmul_pf "matmul_sq__dtype-float32__groups_fit-True__lsize_0-16__lsize_1-16__n-4096__prefetch-True"
cap fd16_8176 finite_diff_strip "finite_diff__dtype-float32__n-8176__tile-16x16"
cap dg_upf_1e6 dg_upf "dg_diff__dtype-float32__nelements-1000000__nmatrices-3__nunit_nodes-64__variant-uPF"
cap dg_nopf_1e6 dg_nopf "dg_diff__dtype-float32__nelements-1000000__nmatrices-3__nunit_nodes-64__variant-noPF"
cap dg_dmpf_1e6 dg_dmpf "dg_diff__dtype-float32__nelements-1000000__nmatrices-3__nunit_nodes-64__variant-dmPF"
cap dg_dmpft_1e6 dg_dmpf "dg_diff__dtype-float32__nelements-1000000__nmatrices-3__nunit_nodes-64__variant-dmPFtrans"
cap dg_tc_64 dg_tc_kernel "dg_diff_tc__dtype-float32__nelements-1000000__nmatrices-3__nunit_nodes-64"
cap dg_tc_48 dg_tc_kernel "dg_diff_tc__dtype-float32__nelements-1000000__nmatrices-3__nunit_nodes-48"
cap dg_tc_32 dg_tc_kernel "dg_diff_tc__dtype-float32__nelements-1000000__nmatrices-3__nunit_nodes-32"
cap dg_tc_16 dg_tc_kernel "dg_diff_tc__dtype-float32__nelements-1000000__nmatrices-3__nunit_nodes-16"
cap dg_tc_128 dg_tc_kernel "dg_diff_tc__dtype-float32__nelements-1000000__nmatrices-3__nunit_nodes-128"
cap madd flops_pattern "flops_madd_pattern__dtype-float32__lid_stride_0-1__lid_stride_1-2048__lsize_0-16__lsize_1-16__m-128__nelements-2097152"
cap tc_8192 matmul_tc "matmul_sq_tc__dtype-float32__lsize_0-16__lsize_1-16__n-8192"
cap gmem2 gmem_pattern "gmem_pattern__dtype-float32__lid_stride_0-1__lid_stride_1-2048__lsize_0-16__lsize_1-16__n_input_arrays-2__nelements-671088640"
cap lmem lmem_shuffle "lmem_shuffle__dtype-float32__lid_stride_0-1__lid_stride_1-2048__lsize_0-16__lsize_1-16__m-1024__nelements-2097152"
cap overlap_m0 overlap "overlap_knl__dtype-float32__lid_stride_0-1__lid_stride_1-2048__lsize_0-16__lsize_1-16__m-0__nelements-268435456"
cap overlap_m8 overlap "overlap_knl__dtype-float32__lid_stride_0-1__lid_stride_1-2048__lsize_0-16__lsize_1-16__m-8__nelements-268435456"
cap fadd flops_pattern "flops_add_pattern__dtype-float32__lid_stride_0-1__lid_stride_1-2048__lsize_0-16__lsize_1-16__m-128__nelements-2097152"
cap barrier barrier_knl "barrier_knl__lid_stride_0-1__lid_stride_1-2048__lsize_0-16__lsize_1-16__m-1024__nelements-2097152"
cap mm_rm_b matmul_rm "matmul_sq_rm__dtype-float32__groups_fit-True__keep-b__lsize_0-16__lsize_1-16__n-4096__prefetch-False"
cap fd_rm_u finite_diff_strip "finite_diff_rm__dtype-float32__keep-u__n-8176__tile-16x16"
cap dg_rm_u dg_rm "dg_diff_rm__dtype-float32__keep-u__nelements-1000000__nmatrices-3__nunit_nodes-64__variant-noPF"
if [ "$only" = "model" ] || [ -z "$only" ]; then
  for k in lm_jobs_kernel eval_points; do
    timeout 600 ncu --set full --clock-control none -k "regex:$k" -c 1 \
      -o $out/ncu_$k -f python tools/run_model_kernels.py > $out/ncu_$k.log 2>&1
    echo "$k rc=$?"
  done
fi
if [ -z "$only" ] || [ "$only" = "launches" ]; then
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 8000 --csv \
  --log-file $out/launches_all.csv python bench.py --steps 1 --warmup 3 --trials-per-step 1 \
  --c5-points 100000 --tc 0 --detail $out/launches_detail.json > $out/launches_bench.log 2>&1
echo "launches rc=$?"
fi
