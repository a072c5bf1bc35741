python tools/sim_ab.py variants/lib_nb2048.so variants/lib_nb1024.so variants/lib_nb512.so variants/lib_nb4096.so variants/lib_nb2048.so 2>&1 | tail -5
