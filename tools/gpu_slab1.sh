# one-barrier fused slab kernel: slab / sharded-step parity, then one GPU's slab timing at N = 1, 2, 4, 8
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_slabstep.py -x -q -k "slab or sharded" 2>&1 | tail -5
for w in 1 2 4 8; do for sync in 2 1; do MQ_PCG_SYNC=$sync python tools/slab_time.py --world $w --iters 60; done; done
