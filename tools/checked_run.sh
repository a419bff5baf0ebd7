# Bound-checked run (the compute-sanitizer substitute; the tool is closed on this
# pool): build the library with -DRCGS_CHECKED into _lib/checked and run the GPU
# suite and the sanitize probe against it.  conftest.py fails the session if any
# device check failed (and checks that a deliberate failure is counted).
set -e
(cd paper_2511_18441_b200/csrc && make -j8 OUT=../_lib/checked/librcgs.so OBJDIR=../_lib/checked/obj EXTRA=-DRCGS_CHECKED >/dev/null)
export RCGS_LIB_PATH=$PWD/paper_2511_18441_b200/_lib/checked/librcgs.so
python -m pytest tests -q -m gpu -s ${PYTEST_ARGS:-} 2>&1 | grep -E "checked build|passed|failed"
python tools/sanitize_probe.py 3
python - <<'PY'
import ctypes, os
lib = ctypes.CDLL(os.environ["RCGS_LIB_PATH"])
c = ctypes.c_uint64(0)
print("sanitize probe: rcgs_debug_violations", lib.rcgs_debug_violations(ctypes.byref(c), 0), c.value)
PY
