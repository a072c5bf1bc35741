timeout 300 python tools/sim_timing.py 2>&1 | tail -6
python tools/sim_ab.py paper_2509_04827_b200/libvoltana.so 2>&1 | tail -1
