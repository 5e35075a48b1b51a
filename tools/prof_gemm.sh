set -u
O=gpurun_out/$1; mkdir -p $O
timeout 300 python -m pytest tests/test_gpu_gemm.py -x -q -m gpu > $O/pytest.log 2>&1; echo rc=$? >> $O/pytest.log
for T in 16 2048; do
timeout 300 ncu --set full --clock-control none --import-source on -k regex:gemm_fused_kernel -s 1 -c 1 -o $O/gemm_fc1_$T -f python tools/gemm_one.py fc1 $T 2 > $O/ncu_$T.log 2>&1
done
