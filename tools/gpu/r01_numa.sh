nvidia-smi topo -m 2>&1 | head -5
lscpu | grep -i numa
cat /sys/bus/pci/devices/$(nvidia-smi --query-gpu=pci.bus_id --format=csv,noheader | head -1 | tr 'A-F' 'a-f' | sed 's/^00000000/0000/')/numa_node 2>&1
for node in 0 1; do cpus=$(lscpu -p=CPU,NODE | grep -v '^#' | awk -F, -v n=$node '$2==n{print $1}' | head -16 | paste -sd,); [ -z "$cpus" ] && continue; echo "node $node cpus $cpus"; taskset -c $cpus python tools/e2e_probe.py 16384 16384 0 2>&1 | grep -E "h2d|d2h|e2e"; done
