mkdir -p gpurun_out
timeout 300 python tools/pcie_bw.py > gpurun_out/pcie_bw.txt 2>&1
