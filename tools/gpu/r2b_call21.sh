# PCIe copy ceilings for the host-buffer e2e path.
O=gpurun_out/r2b21; mkdir -p $O
timeout 300 python tools/pcie_probe.py > $O/pcie.txt 2>&1; cat $O/pcie.txt
nvidia-smi -q | grep -i -A3 "PCIe Generation\|Link Width" | head -20
