"""The public names of the reference package and its modules (nmfa,
nmfa.solver/problem/metrics/gset/generators/kernels) exist here too, so
`import paper_1806_08422_b200 as nmfa` and `from ....solver import X` work as
drop-ins.  The lists were taken from the reference package (pkg/src/nmfa)
with its imported modules and `ThreadPoolExecutor` left out."""

import importlib

import pytest

REFERENCE_NAMES = {
    '': ['AggregateStats', 'DEFAULT_ALPHA', 'DEFAULT_SCHEDULE', 'DEFAULT_SIGMA', 'DEFAULT_TF', 'GroundTruth', 'GsetParseError', 'IsingProblem', 'MAX_EXACT_N', 'NmfaParams', 'RunResult', 'RunStats', 'Schedule', 'Trajectory', 'aggregate', 'brute_force_ground', 'cut_value', 'energy', 'gen_cubic_maxcut', 'gen_dense_maxcut', 'gen_sk', 'generators', 'gset', 'instance_stats', 'is_connected', 'kernels', 'load_gset', 'mean_field', 'median_iqr', 'metrics', 'moebius_ladder', 'nmfa_batch', 'nmfa_run', 'nmfa_step', 'noise_stream', 'normalizers', 'parse_gset', 'problem', 'run_with_noise', 'schedule_eval', 'sign_round', 'solver', 'success_probability', 'time_to_solution', 'write_gset', 'write_results_csv'],
    'solver': ['DEFAULT_ALPHA', 'DEFAULT_SCHEDULE', 'DEFAULT_SIGMA', 'DEFAULT_TF', 'MASK64', 'NmfaParams', 'RUN_STREAM_TAG', 'RunResult', 'Schedule', 'Trajectory', 'dataclass', 'energy', 'nmfa_batch', 'nmfa_run', 'nmfa_step', 'noise_stream', 'replace', 'run_with_noise', 'schedule_eval', 'sign_round'],
    'problem': ['DENSE_THRESHOLD', 'IsingProblem', 'cut_value', 'energy', 'mean_field', 'normalizers', 'sign_round'],
    'metrics': ['AggregateStats', 'ENERGY_TIE_TOL', 'GroundTruth', 'MAX_EXACT_N', 'RunStats', 'aggregate', 'brute_force_ground', 'dataclass', 'instance_stats', 'median_iqr', 'success_probability', 'time_to_solution'],
    'gset': ['GsetParseError', 'IsingProblem', 'RESULT_COLUMNS', 'cut_value', 'load_gset', 'parse_gset', 'write_gset', 'write_results_csv'],
    'generators': ['GEN_STREAM_TAG', 'IsingProblem', 'MASK64', 'gen_cubic_maxcut', 'gen_dense_maxcut', 'gen_sk', 'is_connected', 'moebius_ladder'],
    'kernels': ['BACKEND', 'FORCE_NUMPY', 'anneal_dense', 'anneal_sparse', 'gray_ground'],
}


@pytest.mark.parametrize("module", sorted(REFERENCE_NAMES))
def test_reference_public_names_exist(module):
    mod = importlib.import_module("paper_1806_08422_b200" + ("." + module if module else ""))
    missing = [n for n in REFERENCE_NAMES[module] if not hasattr(mod, n)]
    assert not missing, (module, missing)


# parameter names of the reference's module functions, in order: ours accept the
# same leading parameters (they may add keyword-only or trailing ones)
REFERENCE_SIGNATURES = {
    'generators.gen_cubic_maxcut': ['n', 'seed'],
    'generators.gen_dense_maxcut': ['n', 'p', 'seed'],
    'generators.gen_sk': ['n', 'seed'],
    'generators.is_connected': ['problem'],
    'generators.moebius_ladder': ['n'],
    'gset.load_gset': ['path'],
    'gset.parse_gset': ['text'],
    'gset.write_gset': ['problem'],
    'gset.write_results_csv': ['results', 'metadata'],
    'metrics.aggregate': ['per_instance_stats'],
    'metrics.brute_force_ground': ['problem'],
    'metrics.instance_stats': ['results', 'ground', 'tau_seconds', 'confidence'],
    'metrics.median_iqr': ['values'],
    'metrics.success_probability': ['results', 'ground'],
    'metrics.time_to_solution': ['p', 'tau_seconds', 'confidence'],
    'problem.cut_value': ['problem', 'config'],
    'problem.energy': ['problem', 'config'],
    'problem.mean_field': ['problem', 's'],
    'problem.normalizers': ['problem'],
    'problem.sign_round': ['s'],
    'solver.nmfa_batch': ['problem', 'params', 'n_runs', 'threads', 'record_trajectory'],
    'solver.nmfa_run': ['problem', 'params', 'record_trajectory'],
    'solver.nmfa_step': ['problem', 's', 'T', 'params', 'rng'],
    'solver.noise_stream': ['seed'],
    'solver.run_with_noise': ['problem', 'temps', 'noise', 'alpha', 's0', 'record_trajectory'],
    'solver.schedule_eval': ['schedule', 't', 't_f'],
}


@pytest.mark.parametrize("qualname", sorted(REFERENCE_SIGNATURES))
def test_reference_signatures_are_accepted(qualname):
    import inspect
    module, name = qualname.split(".")
    fn = getattr(importlib.import_module("paper_1806_08422_b200." + module), name)
    ours = [p.name for p in inspect.signature(fn).parameters.values()]
    want = REFERENCE_SIGNATURES[qualname]
    assert ours[:len(want)] == want, (qualname, want, ours)
