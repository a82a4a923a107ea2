mkdir -p gpurun_out
EXP_SHAPES="32768,4096,832" timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_umma_grouped2 -s 3 -c 1 -o gpurun_out/r2e_gemm -f python tools/experiments/exp_gemm.py > gpurun_out/r2e_gemm.log 2>&1; echo "ncu rc=$?"
