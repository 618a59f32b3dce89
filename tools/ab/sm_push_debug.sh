export FSEP_COMM=sm FSEP_SPIN_TIMEOUT_MS=3000
TAG=mix_default timeout 300 python tools/ab/sm_push_debug.py
