timeout 900 python -m paper_1308_1464_b200.benchmatrix --out gpurun_out/matrix_o1.csv > gpurun_out/matrix_o1.log 2>&1; echo rc=$?
timeout 900 python -m paper_1308_1464_b200.benchmatrix --kernels shallow-water-roe euler-hlle euler acoustics-var --sizes 1024x1024 4096x4096 --order 2 --limiter mc --out gpurun_out/matrix_o2.csv > gpurun_out/matrix_o2.log 2>&1; echo rc=$?
tail -3 gpurun_out/matrix_o1.log gpurun_out/matrix_o2.log
