import sys, torch
sys.path.insert(0, ".")
from paper_2310_04734_b200 import assembly, workloads
box, ne = workloads.CFG3_BOX, workloads.CFG3_NE
xyz, conn = assembly.hex27_box(box, *ne)
xd = torch.as_tensor(xyz, device="cuda"); cd = torch.as_tensor(conn, device="cuda")
for _ in range(3):
    Ke, Me = assembly.hex27_helmholtz(xd, cd)
torch.cuda.synchronize()
print("ok")
