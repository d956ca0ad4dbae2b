#!/bin/bash
# One ncu --set full capture per hot-path kernel family (first launch of each),
# summarised into gpurun_out/ncu_all.json by tools/ncu_summary.py.
set -u
cd "$(dirname "$0")/.."
python tools/prof_kernels.py || exit 1
mkdir -p gpurun_out/ncu_all
for k in k_gate_dense k_gate_diag k_swap_indices k_qft_group k_qft_mid k_qft_low4 k_bitrev2 k_tiled k_zgemm_even k_svd_gram_mma_t k_svd_eigen_t k_svd_update_v2 k_swap_regions k_qft_dist_layers k_dist_bitrev k_bitrev_hi; do
  ncu --set full --clock-control none -k regex:"$k" -c 1 -o gpurun_out/ncu_all/$k -f python tools/prof_kernels.py > /dev/null 2>&1
done
python tools/ncu_summary.py gpurun_out/ncu_all/*.ncu-rep > gpurun_out/ncu_all.json
