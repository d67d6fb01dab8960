PIC_DEBUG_SYNC=1 timeout 60 python __graft_entry__.py smoke 2>&1 | grep -v "\[pic\] ok" | tail -12
timeout 900 python -m pytest tests/test_gpu_link.py -q -x --timeout 300 --timeout_method thread -k "not full_width" 2>&1 | tail -40
