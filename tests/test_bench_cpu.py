"""bench.py host logic (CPU): which measured peak the roofline divides by, and the committed DRAM
traffic figure it reports."""
import importlib.util
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _bench():
    spec = importlib.util.spec_from_file_location("bench_under_test", os.path.join(ROOT, "bench.py"))
    m = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(m)
    return m


PEAKS = {"bf16_tflops": 1628.4, "bf16_tflops_sustained": 1374.4}


def test_power_capped_run_uses_the_sustained_peak():
    b = _bench()
    peak, kind = b.select_peak(PEAKS, {"sm_mhz": 1425.0, "sm_max_mhz": 1965.0, "reasons": ["sw_power_cap"]})
    assert peak == 1374.4 and "sustained" in kind
    # clocks well below max with no reason reported also counts as limited
    peak, _ = b.select_peak(PEAKS, {"sm_mhz": 1500.0, "sm_max_mhz": 1965.0, "reasons": []})
    assert peak == 1374.4


def test_full_clock_or_unknown_uses_the_burst_peak():
    b = _bench()
    assert b.select_peak(PEAKS, {"sm_mhz": 1965.0, "sm_max_mhz": 1965.0, "reasons": []})[0] == 1628.4
    assert b.select_peak(PEAKS, None)[0] == 1628.4                       # no clock samples: conservative
    assert b.select_peak({"bf16_tflops": 1628.4}, {"reasons": ["sw_power_cap"]})[0] == 1628.4


def test_profiled_traffic_is_the_committed_capture():
    b = _bench()
    t = b.profiled_traffic("C4", 1)
    assert t is None or 1.5e10 < t < 6e11                                 # >= the algorithmic 15.5 GB
    assert b.profiled_traffic("C4", 8) is None                            # no capture at G = 8


def test_clock_sampler_counts_only_the_timed_window():
    # rows taken before begin() (nvidia-smi start-up, warm-up) and after stop() must not count
    b = _bench()
    c = b.ClockSampler(0)
    row = lambda mhz, cap: [str(mhz), "1965", "900.0", "Not Active", "Not Active", "Not Active", cap]
    c.rows = [row(1965, "Not Active")] * 3
    c.first = len(c.rows)
    c.rows += [row(1400, "Active"), row(1420, "Active")]
    clk = c.stop()
    assert clk["samples"] == 2 and clk["sm_mhz"] == 1410.0 and clk["reasons"] == ["sw_power_cap"]


def test_both_oracle_legs_share_one_sample_definition():
    """cpu_baseline and --impl reference time the same OracleSample (same prompts,
    rows, scaling), so the two legs report the same quantity."""
    import inspect
    b = _bench()
    assert "OracleSample" in inspect.getsource(b.cpu_baseline)
    assert "OracleSample" in inspect.getsource(b.reference_arm)
    from synth import CONFIGS, Workload
    cfg = CONFIGS["C1"]
    w = Workload(cfg, device="cpu")
    P = w.prompts(cfg.N).numpy()
    a = b.cpu_baseline(cfg, w, cfg.N, cfg.M, P, steps=1)
    smp = b.OracleSample(cfg, w, cfg.N, cfg.M, P)
    per, t_sim, t_down = smp.step()
    assert a["kind"] == "oracle" and a["cores"] >= 1 and a["value"] > 0
    assert a["sample"].startswith(smp.describe(t_sim, t_down).split(";")[0])
