python tools/sim_ab.py variants/lib_v4e.so variants/lib_v4e.so 2>&1 | tail -2
