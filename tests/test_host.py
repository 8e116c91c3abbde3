"""CPU-side checks: the C-ABI library, host logic and API surface (no GPU)."""

import ctypes as C
import os
import re

import numpy as np
import pytest

from paper_2108_10591_b200 import _lib, build
from paper_2108_10591_b200.instrument import per_iteration_costs, synthesize
from paper_2108_10591_b200.linalg import CsrMatrix, csr_from_coo, gen_poisson
from paper_2108_10591_b200.problems import CONFIGS, config_stencil, convdiff_stencil, stencil_csr
from paper_2108_10591_b200.reduction import PartitionPlan
from paper_2108_10591_b200.solvers import DeviceEngine, SolverConfig, solve
from tests import golden_cases as gc

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _header_symbols():
    src = open(os.path.join(ROOT, "include", "pbsafe.h")).read()
    return sorted(set(re.findall(r"^\w[\w\s\*]*?\b(pbs_\w+)\s*\(", src, flags=re.M)))


def test_library_builds_and_exports_every_header_symbol():
    path = build.build()
    assert os.path.exists(path)
    lib = C.CDLL(path)
    syms = _header_symbols()
    assert len(syms) >= 15
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    assert sorted(syms) == sorted(_lib.EXPORTS)


def test_sass_is_sm100a():
    import subprocess

    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", build.LIB],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_no_oracle_in_product_package():
    pkg = os.path.join(ROOT, "paper_2108_10591_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                text = open(os.path.join(dirpath, f), encoding="utf-8").read()
                # no import, link or spawn of the checker from product code
                for needle in ("import oracle", "from oracle", "oracle import", "liboracle",
                               "oracle.oracle", "oracle.py", "importlib"):
                    assert needle not in text, (f, needle)


def test_solver_config_validation_matches_reference():
    with pytest.raises(ValueError):
        SolverConfig(tol=0.0)
    with pytest.raises(ValueError):
        SolverConfig(max_iters=0)
    with pytest.raises(ValueError):
        SolverConfig(rr_epoch=0)
    with pytest.raises(ValueError):
        SolverConfig(max_iters=10, rr_cutoff=11)
    with pytest.raises(ValueError):
        SolverConfig(monitor_every=-1)


def test_solve_validates_before_touching_the_device():
    A, _ = gen_poisson(1, 4)
    with pytest.raises(ValueError):
        solve(A, np.ones(4), method="gmres")
    rect = csr_from_coo(2, 3, np.array([0]), np.array([0]), np.array([1.0]))
    with pytest.raises(ValueError):
        solve(rect, np.ones(2))
    with pytest.raises(ValueError):
        solve(A, np.ones(3))
    with pytest.raises(ValueError):
        solve(A, np.ones(4), x0=np.ones(5))
    from paper_2108_10591_b200.linalg import NonFiniteVectorError

    with pytest.raises(NonFiniteVectorError):
        solve(A, np.array([1.0, np.nan, 0.0, 0.0]))
    with pytest.raises(ValueError):
        DeviceEngine(reduce="fastest")


def test_partition_plan_matches_reference_fixture():
    p = np.load(os.path.join(gc.GOLDEN, "plans.npz"))
    pos = 0
    for n, w, ln in zip(p["n"], p["w"], p["lens"]):
        ref = p["bounds"][pos:pos + ln]
        pos += ln
        plan = PartitionPlan.balanced(int(n), int(w))
        got = np.array([lo for lo, _ in plan.ranges] + [plan.ranges[-1][1]])
        assert np.array_equal(got, ref)


@pytest.mark.parametrize("name", gc.case_names())
def test_counter_synthesis_matches_reference(name):
    g = np.load(os.path.join(gc.GOLDEN, f"solve_{name}.npz"))
    spec = dict(__import__("tests.golden._cases", fromlist=["CASES"]).CASES[name])
    iters = int(g["iterations"])
    method = spec["method"]
    replaced = set()
    if method == "pbicgsafe-rr":
        cutoff = spec.get("rr_cutoff") or spec["max_iters"]
        m = spec.get("rr_epoch", 100)
        replaced = {i for i in range(1, iters) if i % m == 0 and i < cutoff}
    # product-type methods: where a breakdown stopped the iteration (the
    # device reports it as stop_stage)
    stage = {"alpha denominator (r0*, Ap)": 1, "omega denominator (At, At)": 2,
             "zeta denominator (At, At)": 2, "zeta/eta denominator e*a - d^2": 2,
             "beta denominator omega": 3, "beta denominator zeta": 3,
             "beta denominator (r0*, r)": 3}.get(str(g["breakdown"]), 0)
    c = synthesize(method, iters, iters < spec["max_iters"], replaced, stop_stage=stage)
    assert c.n_spmv == int(g["n_spmv"])
    assert c.n_dots == int(g["n_dots"])
    assert c.n_reductions == int(g["n_reductions"])


def test_synthesized_costs_match_cost_model():
    c = synthesize("pbicgsafe", 30, True, set())
    row = per_iteration_costs(c, "pbicgsafe")
    assert (row.ax_per_iter, row.dots_per_iter, row.reductions_per_iter) == (2, 9, 1)
    assert (row.scalar_mults_per_iter, row.vec_adds_per_iter, row.workspace_vectors) == (21, 22, 16)
    c = synthesize("ssbicgsafe2", 30, True, set())
    row = per_iteration_costs(c, "ssbicgsafe2")
    assert (row.scalar_mults_per_iter, row.vec_adds_per_iter) == (13, 14)
    # test_instrument.py:32-39, 62-66
    c = synthesize("bicgstab", 30, True, set())
    row = per_iteration_costs(c, "bicgstab")
    assert (row.ax_per_iter, row.dots_per_iter, row.reductions_per_iter) == (2, 5, 2)
    assert (row.scalar_mults_per_iter, row.vec_adds_per_iter, row.workspace_vectors) == (6, 6, 7)
    assert row.tabulated_workspace_vectors == 7
    c = synthesize("gpbicg", 30, True, set())
    row = per_iteration_costs(c, "gpbicg")
    assert (row.ax_per_iter, row.dots_per_iter, row.reductions_per_iter) == (2, 8, 3)


def test_generators_and_config_sizes():
    # SURVEY §8 sizes: C1 n=4096 nnz=20224; C2 nnz=14,581,760 (checked at 16^3 scale here)
    rp, ci, v = stencil_csr(config_stencil("c1"))
    assert len(rp) - 1 == 4096 and rp[-1] == 20224
    k = 16
    rp, ci, v = stencil_csr(convdiff_stencil(3, k, CONFIGS["c2"]["beta"]))
    assert rp[-1] == k**3 + 6 * (k - 1) * k * k
    st = config_stencil("c4", k=8)
    rp, ci, v = stencil_csr(st)
    assert rp[-1] == (3 * 8 - 2) ** 3


def test_csr_matrix_validate():
    A, _ = gen_poisson(2, 5)
    A.validate()
    bad = CsrMatrix(2, 2, np.array([0, 1, 2]), np.array([1, 0]), np.array([1.0, np.inf]))
    from paper_2108_10591_b200.linalg import NonFiniteVectorError

    with pytest.raises(NonFiniteVectorError):
        bad.validate()


def test_pbicgstab_counters_follow_the_oracle_stages():
    """synthesize('pbicgstab', ...) ticks what the oracle's solve_pstab does:
    setup Ax + Ar and one 2-dot batch, then per completed iteration t = A w,
    v = A z and batches of 3 and 5 dots; a stop at stage s ticks the stages
    before it (1 alpha: none, 2 omega: both products + the 3-dot batch,
    3 beta: the x r w update and the 5-dot batch too)."""
    from oracle import oracle as orc
    from paper_2108_10591_b200.instrument import synthesize

    spec, A, b, x0, g = gc.load_case("bs_maxiters5", orc.spmv)
    o = orc.solve(A.row_ptr, A.col_idx, A.values, b, method="pbicgstab", tol=spec["tol"], max_iters=5)
    c = synthesize("pbicgstab", o["iterations"], False, set())
    assert c.n_spmv == o["n_spmv"] == 12
    assert (c.n_dots, c.n_reductions) == (2 + 8 * 5, 1 + 2 * 5)
    for stage, extra_spmv in ((1, 0), (2, 2), (3, 2), (4, 2)):
        c = synthesize("pbicgstab", 3, True, set(), stop_stage=stage)
        assert c.n_spmv == 2 + 2 * 3 + extra_spmv, stage
    o = orc.solve(np.array([0, 1, 2]), np.array([1, 0]), np.array([1.0, 1.0]), np.array([1.0, 0.0]),
                  method="pbicgstab", tol=1e-10, max_iters=10)
    assert o["status"] == "breakdown" and o["failure_iter"] == 0 and o["n_spmv"] == 2
    assert synthesize("pbicgstab", 0, True, set(), stop_stage=1).n_spmv == 2


@pytest.mark.parametrize("bad", [np.nan, np.inf, -np.inf])
@pytest.mark.parametrize("pos", [0, 17, 4095])
def test_check_finite_names_first_bad_index(bad, pos):
    """linalg.py:142-146: the v.v fast path must not hide any non-finite entry,
    and the error names the first bad index."""
    from paper_2108_10591_b200.linalg import NonFiniteVectorError, check_finite

    v = np.random.default_rng(pos).standard_normal(4096)
    v[pos] = bad
    v[-1] = np.nan  # a later bad entry: the first one is reported
    with pytest.raises(NonFiniteVectorError) as ei:
        check_finite(v, "right-hand side")
    assert ei.value.index == pos


def test_check_finite_passes_finite_overflowing_and_empty():
    from paper_2108_10591_b200.linalg import check_finite

    huge = np.full(8, 1e300)  # v.v overflows to inf: the exact scan clears it
    assert check_finite(huge) is huge
    assert check_finite(np.empty(0)).size == 0
    ints = np.arange(5)
    assert check_finite(ints) is ints


def test_bench_reference_arm_contract():
    """bench.py --impl reference: the oracle port of the reference algorithm on
    the host cores prints one JSON line with the driver's keys, the same
    metric / unit / config workload as the device arm, and a cpu_baseline."""
    import json
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    p = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--steps", "1", "--warmup", "3"],
                       cwd=root, capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [ln for ln in p.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["unit"] == "it/s" and d["dtype"] == "f64"
    assert d["value"] > 0 and d["cpu_baseline"]["value"] == d["value"]
    assert d["cpu_baseline"]["kind"] in ("port", "reference") and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["config"]["workload"].startswith("BASELINE config 2")


def test_sass_census_blackwell_async_copies():
    """The hot engines are Blackwell-native in SASS, not just built for sm_100a:
    every staged CSR / sliced-ELL / stencil SpMV instantiation issues 1-D bulk async copies
    (UBLKCP) and waits on mbarrier phases (SYNCS.PHASECHK), and the z-marching
    engine issues 3-D TMA tensor loads (UTMALDG)."""
    import subprocess

    obj = os.path.join(ROOT, "build", "pbsafe", "solve.cu.o")  # the single-GPU schedules' TU
    target = obj if os.path.exists(obj) else build.build()
    sass = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", target], capture_output=True, text=True,
                          timeout=600).stdout
    funcs = {}
    for chunk in re.split(r"\n\s*Function : ", sass)[1:]:
        name, body = chunk.split("\n", 1)
        funcs[name.strip()] = body
    pipe = {n: b for n, b in funcs.items()
            if "csr_pipe_kernel" in n or "stencil_pipe_kernel" in n or "sell_pipe_kernel" in n}
    zm = {n: b for n, b in funcs.items() if "stencil_zm_kernel" in n}
    sell = [n for n in pipe if "sell_pipe_kernel" in n]
    assert len(pipe) >= 20 and len(zm) >= 8 and len(sell) >= 18, (len(pipe), len(zm), len(sell))
    for n, b in pipe.items():
        assert "UBLKCP" in b and "SYNCS.PHASECHK" in b, n
    for n, b in zm.items():
        assert "UTMALDG" in b and "SYNCS.PHASECHK" in b, n
    # the two kernels of the config-2 iteration and the config-4 matrix-free K12
    # (sliced-ELL K12 / K3 in the pair-dictionary mode, 2 CTAs per SM; the CSR-order pair; z-marching K12)
    hot = ("sell_pipe_kernelINS_7EpiK12TILb1EEELi2ELi2E", "sell_pipe_kernelINS_6EpiK3TILj77EEELi2ELi2E",
           "csr_pipe_kernelINS_7EpiK12TILb1EEE", "csr_pipe_kernelINS_6EpiK3TILj77EEE",
           "stencil_zm_kernelINS_7EpiK12TILb1EEELi27E")
    for h in hot:
        assert any(h in n for n in funcs), h


def test_bench_gpus_n_self_launches_n_ranks():
    """bench.py --gpus N without torchrun's environment re-launches itself
    under torch.distributed.run with N processes; every rank reaches the
    rendezvous and rank 0's line reports n_gpus = N (dry run: no GPU work)."""
    import json
    import subprocess
    import sys

    p = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--config", "c4", "--dry-run"], cwd=ROOT,
                       capture_output=True, text=True, timeout=300,
                       env={k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")})
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [ln for ln in p.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1, p.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["schedule"] == "partitioned" and d["config"] == "c4"


def test_bench_rejects_world_size_mismatch():
    import subprocess
    import sys

    env = {**os.environ, "WORLD_SIZE": "2", "RANK": "0", "LOCAL_RANK": "0"}
    p = subprocess.run([sys.executable, "bench.py", "--gpus", "4", "--dry-run"], cwd=ROOT, capture_output=True,
                       text=True, timeout=120, env=env)
    assert p.returncode != 0 and "WORLD_SIZE=2" in (p.stderr + p.stdout)
