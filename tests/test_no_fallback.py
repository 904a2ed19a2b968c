"""The product path has no CPU or oracle fallback (CPU tests): a missing libmoe.so fails the
import (CPU tensors are rejected: tests/test_abi.py), and nothing in the package imports the
oracle (only tests/, __graft_entry__.smoke() and bench.py's CPU arms may)."""
import ast
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2605_05049_b200")


def test_missing_library_fails_the_import():
    env = {**os.environ, "MOE_LIB": os.path.join(ROOT, "does_not_exist", "libmoe.so")}
    p = subprocess.run([sys.executable, "-c", "import paper_2605_05049_b200"], cwd=ROOT, env=env,
                       capture_output=True, text=True, timeout=300)
    assert p.returncode != 0
    assert "ImportError" in p.stderr or "OSError" in p.stderr


def test_package_never_imports_the_oracle():
    for dirpath, _, files in os.walk(PKG):
        for fn in files:
            if not fn.endswith(".py"):
                continue
            tree = ast.parse(open(os.path.join(dirpath, fn)).read())
            for node in ast.walk(tree):
                names = []
                if isinstance(node, ast.Import):
                    names = [a.name for a in node.names]
                elif isinstance(node, ast.ImportFrom):
                    names = [node.module or ""]
                assert not any(n == "oracle" or n.startswith("oracle.") for n in names), (fn, names)
