"""Paper integers of the workload definition and weak-scaling normalisation.

Table II: circuits = 2 (n+1) L^2; rho = circuits_per_gpu / 3755;
t_norm = t_actual * N_actual / N_ideal; efficiency 61.85 / 64.92 = 95.3 %.
"""

from conftest import golden


def test_circuit_counts_table2():
    g = golden("table2.json")
    for row in g["rows"]:
        assert 2 * (g["n"] + 1) * row["L"] ** 2 == row["circuits"]
        assert round(row["circuits"] / row["gpus"]) == row["circuits_per_gpu"]


def test_rho_and_tnorm_table2():
    g = golden("table2.json")
    base = g["baseline_circuits_per_gpu"]
    for row in g["rows"]:
        rho = row["circuits"] / row["gpus"] / base
        assert abs(rho - row["rho"]) <= 0.005 * max(row["rho"], 0.02) + 5e-4
        n_ideal = row["circuits"] / base
        t_norm = row["t_actual"] * row["gpus"] / n_ideal if rho < 1 else row["t_actual"]
        assert abs(t_norm - row["t_norm"]) <= 0.005 * row["t_norm"]


def test_weak_scaling_efficiency():
    g = golden("table2.json")
    eff = 100 * g["rows"][4]["t_actual"] / g["rows"][5]["t_actual"]
    assert abs(eff - g["weak_scaling_efficiency_pct"]) < 0.1
