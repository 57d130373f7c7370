out=gpurun_out/s2v; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_sessions.py tests/test_gpu_ops.py tests/test_gpu_edge.py tests/test_formats.py -x -q > $out/pytest.txt 2>&1; echo "exit $?" >> $out/pytest.txt
PROBE_JOBS=2 timeout 600 python tools/upload_probe.py c2 > $out/up_pinned.txt 2>&1
PROBE_JOBS=2 PROBE_PAGEABLE=1 timeout 900 python tools/upload_probe.py c2 > $out/up_pageable.txt 2>&1
PROBE_JOBS=2 PROBE_PAGEABLE=1 FL_NO_STAGED_COPY=1 timeout 900 python tools/upload_probe.py c2 > $out/up_pageable_nostage.txt 2>&1
tail -2 $out/pytest.txt; grep job $out/up_*.txt
