cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests/test_fuselage_gpu.py tests/test_linalg_gpu.py tests/test_dist_gpu.py tests/test_fdm_gpu.py tests/test_mor_gpu.py tests/test_greedy_gpu.py -q -m gpu --timeout 600 2>&1 | tail -15
timeout 600 python tools/prof_orth.py
python tools/rom_accuracy.py --configs cfg3 --points 30,70,110,150,185,215,240,262,282,298 --moments 5 --stride 5
python tools/rom_accuracy.py --configs cfg3 --points 35,80,125,165,200,230,255,277,296 --moments 5 --stride 5
python tools/rom_accuracy.py --configs cfg2 --points 40,100,160,220,280,330,380,420,460,495 --moments 6 --stride 5
python tools/rom_accuracy.py --configs cfg2 --points 30,80,130,180,230,280,330,370,410,445,475,498 --moments 5 --stride 5
python tools/rom_accuracy.py --configs cfg2 --greedy --moments 6 --max-points 14 --stride 5
