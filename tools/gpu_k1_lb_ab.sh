#!/bin/bash
# K1 flush-group A/B (variants/<v>.so): GPU device suite on the candidates, then K1 time per density
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
for v in ${TEST_VARIANTS:-}; do PULSE_LIB=$PWD/variants/$v.so timeout 600 python -m pytest tests/test_gpu_device.py -m gpu -q -x -p no:cacheprovider 2>&1 | tail -1; done
for sp in ${SPS:-0.9 0.95 0.99}; do for v in ${VARIANTS:-lb4}; do echo -n "$v "; PULSE_LIB=$PWD/variants/$v.so timeout 300 python tools/k1_time.py $sp 2>&1 | tail -1; done; done
