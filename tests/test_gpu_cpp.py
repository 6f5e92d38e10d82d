import subprocess

import pytest

from tests.test_abi import _compile_client

pytestmark = pytest.mark.gpu


def test_cpp_client_runs(gk, tmp_path):
    exe = _compile_client(str(tmp_path / "client"))
    r = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stderr
    lines = r.stdout.strip().splitlines()
    assert lines[0].startswith("(0, 0)") and "erased 10, live 99990" in lines[-1]
