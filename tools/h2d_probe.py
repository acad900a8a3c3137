"""H2D bandwidth from pinned host memory with the process bound to each NUMA node."""
import os, time, glob
import torch
props = torch.cuda.get_device_properties(0)
bus = getattr(props, "pci_bus_id", None)
print("pci", getattr(props, "pci_domain_id", None), bus, getattr(props, "pci_device_id", None))
nodes = sorted(glob.glob("/sys/devices/system/node/node[0-9]*"))
print("numa nodes", [os.path.basename(n) for n in nodes])
for dev in glob.glob("/sys/bus/pci/devices/*"):
    try:
        if open(dev + "/vendor").read().strip() == "0x10de" and open(dev + "/class").read().startswith("0x0302"):
            print(dev, "numa_node", open(dev + "/numa_node").read().strip())
    except Exception:
        pass
allcpu = os.sched_getaffinity(0)
def cpus(node):
    out = set()
    for part in open(node + "/cpulist").read().strip().split(","):
        a, _, b = part.partition("-")
        out.update(range(int(a), int(b or a) + 1))
    return out
for node in nodes + [None]:
    os.sched_setaffinity(0, cpus(node) if node else allcpu)
    h = torch.empty(4 << 30, dtype=torch.uint8, pin_memory=True)
    h.fill_(1)
    d = torch.empty_like(h, device="cuda")
    for _ in range(2):
        torch.cuda.synchronize(); t0 = time.perf_counter(); d.copy_(h, non_blocking=True); torch.cuda.synchronize(); t1 = time.perf_counter()
    print(os.path.basename(node) if node else "all", "%.1f GB/s" % (h.numel() / (t1 - t0) / 1e9), flush=True)
    del h, d
    torch.cuda.empty_cache()
