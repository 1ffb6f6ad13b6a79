# The reference's own test suite against this package on the GPU (host-mirror
# mode; stage it first in the build container: python scripts/reference_suite.py stage)
timeout 1800 python scripts/reference_suite.py run > gpurun_out/reference_suite.log 2>&1
tail -5 gpurun_out/reference_suite.log
