timeout 300 python tools/adamw_probe.py 2>&1 | tail -6
timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_nn.py -x -q --timeout 600 -k "adamw or optim or Adam" 2>&1 | tail -2
cp paper_2511_05811_b200/_build/libmoss_b200.so /tmp/new.so; cp paper_2511_05811_b200/_build/libmoss_old.so paper_2511_05811_b200/_build/libmoss_b200.so
echo "--- previous kernel"; timeout 300 python tools/adamw_probe.py 2>&1 | tail -6
cp /tmp/new.so paper_2511_05811_b200/_build/libmoss_b200.so
