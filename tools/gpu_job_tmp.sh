mkdir -p gpurun_out
timeout 300 python tools/pcie_bw.py > gpurun_out/pcie.txt 2>&1; cat gpurun_out/pcie.txt
timeout 600 python tools/e2e_probe.py > gpurun_out/e2e_probe.txt 2>&1; cat gpurun_out/e2e_probe.txt
