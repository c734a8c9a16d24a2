mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 300 python scripts/v1_probe.py vgg16 256 > gpurun_out/v1_probe256_mbar.json 2>&1; cat gpurun_out/v1_probe256_mbar.json | cut -c1-400
timeout 900 compute-sanitizer --tool racecheck --error-exitcode 17 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "test_v1_containers_bit_exact or general_alphabet_containers" > gpurun_out/racecheck_v1.log 2>&1; echo "racecheck rc=$?"; tail -4 gpurun_out/racecheck_v1.log
