timeout 400 python tools/prefill_points.py 8192,28672,2.5,64 8192,28672,2.5,256 8192,28672,2.5,2048 28672,8192,2.5,2048 1024,4096,3.25,2048 8192,28672,3.0,4096 2>&1 | tail -7
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 8 --csv python tools/prefill_points.py 8192,28672,2.5,2048 2>/dev/null | grep -v "^==" | awk -F'","' '{print $5, $NF}' | cut -c1-40,150-200
