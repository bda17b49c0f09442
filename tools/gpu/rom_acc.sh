cd $GRAFT_REPO_ROOT
python tools/rom_accuracy.py --configs cfg2 cfg3 --stride 5
python tools/rom_accuracy.py --configs cfg2 --points 40,100,160,220,280,330,380,420,460,495 --moments 6 --stride 5
python tools/rom_accuracy.py --configs cfg3 --points 35,85,130,170,205,235,260,280,295 --moments 6 --stride 5
python tools/rom_accuracy.py --configs cfg2 --greedy --moments 6 --max-points 14 --stride 5
python tools/rom_accuracy.py --configs cfg3 --greedy --moments 5 --max-points 14 --stride 5
