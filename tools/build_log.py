"""Verbose nvcc build of libsor into a scratch path; writes the ptxas log (development aid)."""
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1401_0763_b200 import build as B  # noqa: E402

out = sys.argv[1] if len(sys.argv) > 1 else "/tmp/libsor_test.so"
log = sys.argv[2] if len(sys.argv) > 2 else "/tmp/build.log"
nc = B.nccl_dir()
cmd = [B.NVCC, *B.NVCC_FLAGS, "-Xptxas=-v", *("-D" + d for d in sys.argv[3:]), "-I" + B.INCLUDE,
       "-I" + os.path.join(nc, "include"), os.path.join(B.CSRC, "sor_api.cu"), "-o", out,
       "-L" + os.path.join(nc, "lib"), "-l:libnccl.so.2", "-Xlinker", "-rpath=" + os.path.join(nc, "lib")]
r = subprocess.run(cmd, capture_output=True, text=True)
open(log, "w").write(r.stderr + r.stdout)
print("rc", r.returncode)
if r.returncode:
    print(r.stderr[-3000:])
