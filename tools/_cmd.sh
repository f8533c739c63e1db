S2D_LIB_PATH=$PWD/paper_2604_03092_b200/lib/diag/libsurfel2d.so python tools/diag_stats.py
bash tools/ab.sh default un2
