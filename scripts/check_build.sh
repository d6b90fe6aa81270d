# Device-side bounds-check build (XFLAGS=-DSGDB_CHECKS: asserts on the model /
# coefficient-slice gathers, coefficient and partial-sum stores, row-block
# geometry and the one-launch step's release counts; kernels_sparse.cu) and the
# sparse full-batch / sync GPU suites run against it. compute-sanitizer is not
# available on the GPU pool; a failed check traps the kernel (cudaErrorAssert)
# and fails the test.
#   here:        bash scripts/check_build.sh build
#   on the box:  bash scripts/check_build.sh run   (log: gpurun_out/check_build_tests.txt)
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
if [ "$1" = build ]; then
  make -C "$ROOT/paper_1802_08800_b200/csrc" -j8 OUT="$ROOT/checks/libsgdb_b200.so" BUILD="$ROOT/build/checks" XFLAGS=-DSGDB_CHECKS
  exit 0
fi
LIB="$ROOT/paper_1802_08800_b200/libsgdb_b200.so"
cp "$LIB" /tmp/libsgdb_b200.release.so
cp "$ROOT/checks/libsgdb_b200.so" "$LIB"
mkdir -p "$ROOT/gpurun_out"
set +e
timeout 1200 python -m pytest -q -p no:cacheprovider tests/test_gpu_segments.py tests/test_gpu_sync.py \
  tests/test_gpu_configs.py tests/test_gpu_nccl.py tests/test_gpu_golden.py > "$ROOT/gpurun_out/check_build_tests.txt" 2>&1
rc=$?
cp /tmp/libsgdb_b200.release.so "$LIB"
echo "check build tests rc=$rc" >> "$ROOT/gpurun_out/check_build_tests.txt"
exit $rc
