#!/bin/bash
# Host topology of the GPU box: cores, NUMA nodes, the GPU's NUMA node, memory.
echo "nproc=$(nproc)"; lscpu | egrep "Model name|Socket|Core|Thread|NUMA|L3" ; 
for n in /sys/devices/system/node/node*; do echo "$n cpus=$(cat $n/cpulist) mem=$(grep MemTotal $n/meminfo)"; done
nvidia-smi --query-gpu=pci.bus_id,name,memory.total --format=csv
python - <<'PY'
import torch, os
p = torch.cuda.get_device_properties(0)
bdf = "%04x:%02x:%02x.0" % (p.pci_domain_id, p.pci_bus_id, p.pci_device_id)
print("bdf", bdf, "numa_node", open("/sys/bus/pci/devices/%s/numa_node" % bdf).read().strip(),
      "affinity", len(os.sched_getaffinity(0)), "total_memory", p.total_memory)
PY
free -g
