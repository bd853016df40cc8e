for v in "$@"; do
  touch paper_1911_02373_b200/csrc/rp_gram.cu
  make -s -C paper_1911_02373_b200/csrc EXTRA="$v" > /dev/null 2>&1 || { echo "$v: build failed"; continue; }
  echo "$v: $(timeout 120 python tools/prof_kernels.py gram --reps 10)"
done
touch paper_1911_02373_b200/csrc/rp_gram.cu
