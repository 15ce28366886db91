mkdir -p gpurun_out
for lib in _ablibs/head.so _ablibs/work.so; do SSB_LIB=$lib timeout 600 python scripts/c5_concurrency.py; done > gpurun_out/conc.log 2>&1
