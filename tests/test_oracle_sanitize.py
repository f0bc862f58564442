"""The C oracle under AddressSanitizer + UndefinedBehaviorSanitizer (host oracle built
with -fsanitize=address,undefined): tests/native/oracle_sanitize_main.c drives every algorithm,
optimizer, shaping and bound variant, the ranking corner cases (ties, NaN, ±0, ±inf, N = 1) and
the MLP problem; any invalid access or undefined operation aborts the run."""
import os
import shutil
import subprocess
import tempfile

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.skipif(shutil.which("gcc") is None, reason="gcc not available")
def test_oracle_under_asan_ubsan():
    with tempfile.TemporaryDirectory() as td:
        exe = os.path.join(td, "orc_san")
        cmd = ["gcc", "-std=c11", "-O1", "-g", "-fno-omit-frame-pointer",
               "-fsanitize=address,undefined", "-fno-sanitize-recover=all",
               "-I", os.path.join(ROOT, "oracle"), os.path.join(ROOT, "oracle", "es_oracle.c"),
               os.path.join(ROOT, "tests", "native", "oracle_sanitize_main.c"), "-o", exe, "-lm"]
        b = subprocess.run(cmd, capture_output=True, text=True)
        if b.returncode != 0 and "asan" in (b.stderr or "").lower():
            pytest.skip("sanitizer runtime unavailable: " + b.stderr[-200:])
        assert b.returncode == 0, b.stderr
        env = dict(os.environ, ASAN_OPTIONS="detect_leaks=1:abort_on_error=0",
                   UBSAN_OPTIONS="print_stacktrace=1")
        r = subprocess.run([exe], capture_output=True, text=True, env=env, timeout=300)
        assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stdout + r.stderr
