timeout 600 python tools/frame_probe.py 2>&1 | head -40
