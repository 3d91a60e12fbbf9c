# Build libforkkv variants of ra_tc.cu with extra -D flags (diagnostic A/B timing on the GPU box):
#   bash tools/variants.sh name "-DFOO=1" ...   -> paper_2604_06370_b200/variants/libforkkv_<name>.so
# select one at run time with FKV_LIB_PATH=paper_2604_06370_b200/variants/libforkkv_<name>.so
set -e
cd "$(dirname "$0")/.."
python -m paper_2604_06370_b200.build > /dev/null
objs=$(python - <<'PY'
import os
from paper_2604_06370_b200 import build as b
for src in b._sources():
    if os.path.basename(src) == "ra_tc.cu":
        continue
    name = os.path.splitext(os.path.basename(src))[0] + os.path.splitext(src)[1].replace(".", "_")
    print(os.path.join(b.OBJ, f"{name}.{b._digest(src)}.o"))
PY
)
mkdir -p paper_2604_06370_b200/variants /tmp/fkv_var
names=""
while [ $# -gt 0 ]; do
  name=$1; flags=$2; shift 2
  names="$names $name"
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC \
    -Iinclude -Ipaper_2604_06370_b200/csrc $flags -c paper_2604_06370_b200/csrc/ra_tc.cu -o /tmp/fkv_var/ra_tc_$name.o &
done
wait
for name in $names; do
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -Xcompiler -fPIC -cudart static \
    -o paper_2604_06370_b200/variants/libforkkv_$name.so /tmp/fkv_var/ra_tc_$name.o $objs
  echo built $name
done
