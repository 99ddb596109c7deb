set -x
nproc; lscpu | head -30; free -g; cat /sys/kernel/mm/transparent_hugepage/enabled; cat /sys/kernel/mm/transparent_hugepage/defrag; numactl -H 2>/dev/null | head; nvidia-smi topo -m; nvidia-smi -q | grep -i -A3 "pci\b\|Link Width\|Link Gen" | head -40
./tools/probe/pin_probe_bin 16
