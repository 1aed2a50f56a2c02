"""cProfile of the Python machine on the GPU box (all threads via
threading.setprofile is too heavy; profile the single-worker case)."""
import cProfile
import pstats
import sys

sys.path.insert(0, ".")
from paper_2303_08058_b200.bridge import IntegrationMode  # noqa: E402
from paper_2303_08058_b200.cli import RunConfig, run_single  # noqa: E402

cfg = RunConfig(subgrids=512, steps=2, repeats=1, workers=1, executors=32, max_agg=8,
                integration=IntegrationMode.POLLING, warmup_steps=1)
res = run_single(cfg)
print("W1 ms/step", [round(x, 1) for x in res.step_ms])
cfg8 = RunConfig(subgrids=512, steps=3, repeats=1, workers=8, executors=32, max_agg=8,
                 integration=IntegrationMode.POLLING, warmup_steps=1)
print("W8 ms/step", [round(x, 1) for x in run_single(cfg8).step_ms])
cProfile.run("run_single(cfg)", "/tmp/pm.prof")
st = pstats.Stats("/tmp/pm.prof")
st.sort_stats("tottime").print_stats(25)
