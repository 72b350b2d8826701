CF_RING_CHAIN=0 timeout 300 python tools/c1_ring_probe.py > gpurun_out/c1ring_chain0.log 2>&1
CF_RING_CHAIN=1 timeout 300 python tools/c1_ring_probe.py > gpurun_out/c1ring_chain1.log 2>&1
