lscpu | grep -i "numa\|^CPU(s)\|Model name"
B=$(nvidia-smi --query-gpu=pci.bus_id --format=csv,noheader | head -1 | tr 'A-Z' 'a-z' | sed 's/^0000//; s/^/0000/')
echo "gpu bus $B"; cat /sys/bus/pci/devices/${B#0000}/numa_node 2>/dev/null; ls /sys/bus/pci/devices/ | grep -i "${B: -7}" ; cat /sys/bus/pci/devices/*${B: -10}/numa_node 2>/dev/null
which taskset numactl
cat /proc/self/status | grep Cpus_allowed_list
