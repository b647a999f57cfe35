# the fused peer-memory exchange (isr_peer.cuh) on one GPU through the halo loopback: exchange tests (both transports), graph loop, capacity growth
timeout 900 python -m pytest tests/test_gpu_exchange.py -q -x > gpurun_out/peer_tests.log 2>&1; echo "exchange tests rc=$?"; tail -15 gpurun_out/peer_tests.log
