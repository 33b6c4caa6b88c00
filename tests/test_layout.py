"""Repository layout rules (task ③/⑥).

* the product package never imports, links or loads anything under oracle/
  (the oracle is the checker, never the thing measured or shipped);
* the product has no CPU compute fallback: every compute entry point goes
  through libtbf_b200.so;
* nothing the GPU box runs reads /root/reference at run time.
"""
import ast
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2411_03029_b200")


def _py_files(d):
    for dp, _, fs in os.walk(d):
        if "_build" in dp or "__pycache__" in dp:
            continue
        for f in fs:
            if f.endswith(".py"):
                yield os.path.join(dp, f)


def test_product_never_imports_oracle():
    for path in _py_files(PKG):
        tree = ast.parse(open(path).read(), path)
        for node in ast.walk(tree):
            if isinstance(node, ast.Import):
                names = [a.name for a in node.names]
            elif isinstance(node, ast.ImportFrom):
                names = [node.module or ""]
            else:
                continue
            for n in names:
                assert not n.split(".")[0] == "oracle", f"{path} imports {n}"
        src = open(path).read()
        assert "liboracle" not in src and "libref" not in src, path


def test_native_sources_do_not_reference_oracle():
    for dp, _, fs in os.walk(os.path.join(PKG, "csrc")):
        for f in fs:
            src = open(os.path.join(dp, f)).read()
            assert not re.search(r"#include\s+[\"<][^\">]*oracle", src), f
            assert "/root/reference" not in src, f


def _code_strings(tree):
    """String literals that are not docstrings (docstrings may cite ref files)."""
    docs = set()
    for node in ast.walk(tree):
        if isinstance(node, (ast.Module, ast.FunctionDef, ast.ClassDef, ast.AsyncFunctionDef)):
            if node.body and isinstance(node.body[0], ast.Expr) and isinstance(node.body[0].value, ast.Constant):
                docs.add(id(node.body[0].value))
    for node in ast.walk(tree):
        if isinstance(node, ast.Constant) and isinstance(node.value, str) and id(node) not in docs:
            yield node.value


def test_no_runtime_reads_of_reference():
    # bench.py, the product package and smoke() must not depend on /root/reference
    for path in [os.path.join(ROOT, "bench.py")] + list(_py_files(PKG)):
        for sv in _code_strings(ast.parse(open(path).read())):
            assert "/root/reference" not in sv, path
    ge = open(os.path.join(ROOT, "__graft_entry__.py")).read()
    smoke = next(n for n in ast.parse(ge).body if isinstance(n, ast.FunctionDef) and n.name == "smoke")
    for sv in _code_strings(smoke):
        assert "/root/reference" not in sv


def test_bench_uses_oracle_only_in_cpu_legs():
    src = open(os.path.join(ROOT, "bench.py")).read()
    tree = ast.parse(src)
    allowed = {"cpu_baseline", "run_reference", "_cpu_baseline", "cpu_port_baseline"}
    for fn in tree.body:
        if not isinstance(fn, ast.FunctionDef):
            continue
        seg = ast.get_source_segment(src, fn)
        if re.search(r"\bfrom oracle\b|\bimport oracle\b", seg):
            assert fn.name in allowed, f"bench.py:{fn.name} imports the oracle"
