# GEMM-kernel-only durations (ncu launch list) of CTA-pair tiles with split K at the qkvA / dA shapes
nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++20 -I include tools/gemm_bench.cu -o /tmp/gemm_bench -L paper_2605_08314_b200 -lfsvd_b200 -Xlinker -rpath=$PWD/paper_2605_08314_b200 || exit 1
for shp in "512 3687 4096" "512 1791 11008" "512 12288 1229"; do
for cfg in "128 1 1 1" "256 1 1 2" "256 1 2 2" "256 1 3 2" "256 1 4 2" "256 2 2 2" "256 2 4 2" "256 1 2 1" "256 2 2 1"; do
  set -- $cfg
  echo "== $shp BN=$1 BMT=$2 SPLITS=$3 CG=$4"
  FSVD_GEMM_BN=$1 FSVD_GEMM_BMT=$2 FSVD_GEMM_SPLITS=$3 FSVD_GEMM_CG=$4 timeout 120 ncu --metrics gpu__time_duration.sum --clock-control none --csv /tmp/gemm_bench $shp 3 2>/dev/null | grep -E "gemm_tc_kernel|splitk" | awk -F'","' '{print $5 " " $NF}' | sed 's/"//g' | sort | uniq -c | head -4
done
done
