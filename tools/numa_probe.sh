nvidia-smi topo -m 2>&1 | head -20
ls /sys/devices/system/node/ | head; cat /sys/devices/system/node/node*/cpulist 2>/dev/null
nproc; python - <<'PY'
import os, torch, time
print("affinity", len(os.sched_getaffinity(0)))
dev = torch.cuda.get_device_properties(0)
print(dev.name, torch.cuda.get_device_properties(0).pci_bus_id if hasattr(dev,'pci_bus_id') else '')
PY
cat /sys/bus/pci/devices/*/numa_node 2>/dev/null | sort | uniq -c
for f in /sys/bus/pci/drivers/nvidia/0000:*; do echo $f $(cat $f/numa_node) $(cat $f/local_cpulist); done
