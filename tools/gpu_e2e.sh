# host-API tests + the bench's e2e leg (stage laps with PULSE_TIMING=1)
timeout 900 python -m pytest tests/test_host_api.py tests/test_cpp_api.py tests/test_resident.py -q 2>&1 | tail -2
PULSE_TIMING=1 timeout 900 python bench.py --no-cpu-baseline --steps 3 > gpurun_out/e2e_bench.json 2> gpurun_out/e2e_bench.err; echo "bench rc=$?"
python -c "import json; d=json.loads(open('gpurun_out/e2e_bench.json').read().strip().split(chr(10))[-1]); print(d['e2e'])"
grep -E "decode|read_patch|write_patch|encode" gpurun_out/e2e_bench.err | tail -30
