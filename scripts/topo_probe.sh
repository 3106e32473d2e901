set -x
nvidia-smi topo -m
nvidia-smi --query-gpu=index,pci.bus_id --format=csv
lscpu | head -30
for d in /sys/bus/pci/devices/*; do if [ -f $d/class ] && grep -q 0x030200 $d/class; then echo $d $(cat $d/numa_node) $(cat $d/local_cpulist); fi; done
cat /proc/self/status | grep -i allowed
which numactl taskset
nproc
