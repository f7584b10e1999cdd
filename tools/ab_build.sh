#!/bin/bash
# A/B builds of libspmat with spmv.cu compiled under extra -D flags:
#   tools/ab_build.sh NAME -DFOO=1 ...   ->  paper_2406_08646_b200/_ab/NAME.so
# run with SPMAT_LIB=paper_2406_08646_b200/_ab/NAME.so
set -e
name=$1; shift
python -m paper_2406_08646_b200.build >/dev/null
python - "$name" "$@" <<'PY'
import os, subprocess, sys
import paper_2406_08646_b200.build as b
name, extra = sys.argv[1], sys.argv[2:]
out = os.path.join(b.HERE, "_ab"); os.makedirs(out, exist_ok=True)
obj = os.path.join(out, name + "_spmv.o")
subprocess.run([b.nvcc(), "-c", os.path.join(b.CSRC, "spmv.cu"), "-o", obj] + b._flags() + extra, check=True, capture_output=True)
objs = [obj if s == "spmv.cu" else os.path.join(b.OBJ, s.replace(".cu", ".o")) for s in b.SOURCES]
subprocess.run([b.nvcc(), "-shared", "-o", os.path.join(out, name + ".so")] + objs + b.ARCH + ["-ldl"], check=True)
print(os.path.join(out, name + ".so"))
PY
