cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python tools/ab_variants.py shipped:SGKKT_GRID9=1 pf0:SGKKT_GRID9=1 pf4:SGKKT_GRID9=1 shipped:SGKKT_GRID9=1,SGKKT_GRID_SEG=32 shipped:SGKKT_GRID9=1,SGKKT_GRID_SEG=43 shipped:SGKKT_GRID9=1,SGKKT_GRID_SEG=85 shipped:SGKKT_GRID9=1,SGKKT_GRID_SEG=128 shipped:SGKKT_GRID9=1,SGKKT_GRID_SEG=255 > gpurun_out/g57_ab.log 2>&1
cat gpurun_out/g57_ab.log
python -c "
from paper_2512_23804_b200.device import _grid_seg_len
print('default seg', _grid_seg_len(255, 65025))"
