which=$1; envs=$2; shift 2
for v in "$@"; do
  touch paper_1911_02373_b200/csrc/*.cu
  make -s -C paper_1911_02373_b200/csrc EXTRA="$v" > /dev/null 2>&1 || { echo "$v: build failed"; continue; }
  echo "$v: $(env $envs timeout 300 python tools/prof_kernels.py $which --reps 3 2>&1 | tail -1)"
done
