for wd in 16 32 64 128; do SLAB_WIDTH=$wd python tools/slab_parts.py 4 1 4 8; done > gpurun_out/slab_w_c4.log 2>&1
