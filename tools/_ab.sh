for l in cur scam scam5 cur5; do DIVAS_LIB=_variants/$l.so python tools/time_fuse.py --config C3 --iters 30; done > gpurun_out/ab32.log 2>&1
