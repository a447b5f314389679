bash scripts/official.sh
bash scripts/configs_all.sh
python tools/e2e_timeline.py > gpurun_out/e2e_tl.txt 2>&1
python tools/pcie_copy.py > gpurun_out/pcie.txt 2>&1
