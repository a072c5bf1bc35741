python tools/sim_ab.py paper_2509_04827_b200/libvoltana.so 2>&1 | tail -1
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -3
