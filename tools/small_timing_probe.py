"""Phase timestamps of the one-launch small path on c1 (development tool): build the timing variant
with FMM_BUILD_VARIANT=stime FMM_EXTRA_FLAGS=-DFMM_SMALL_TIMING python paper_1409_2908_b200/build.py, then
FMM_LIB_PATH=paper_1409_2908_b200/libfmm_stime.so python tools/small_timing_probe.py [L] (device printf per launch)."""
import os, sys, torch
sys.path.insert(0, os.getcwd())
import paper_1409_2908_b200 as F
L = int(sys.argv[1]) if len(sys.argv) > 1 else 1
A = torch.rand(256, 256, dtype=torch.float64, device="cuda"); B = torch.rand(256, 256, dtype=torch.float64, device="cuda")
p = F.Plan(F.load_alg("strassen_222_7"), 256, 256, 256, L)
C = p.new_output()
for i in range(5):
    p.execute(A, B, C)
    torch.cuda.synchronize()
    print("----", flush=True)
