"""cfg3 multi-RHS (W = 900) matvec time: median of 5 after 2 warm-ups (CUDA events)."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_20350_b200.problems import seeded_stacked4, system_from_generator, unit_feed_rhs  # noqa
from paper_2506_20350_b200.solvers import BorderedOperator  # noqa
from paper_2506_20350_b200.toeplitz import generator_from_stacked, matvec  # noqa

op = BorderedOperator.from_system(system_from_generator(generator_from_stacked(seeded_stacked4(30, 30, 256, 0))))
B = torch.from_numpy(unit_feed_rhs(30, 30, 256, columns="each")).cuda()
for _ in range(2):
    matvec(op.spectral, B)
ts = []
for _ in range(5):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); matvec(op.spectral, B); e1.record(); torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
print(os.environ.get("TOEP_FFT_STREAM", "-"), os.environ.get("TOEP_FFT_STREAM_TIL", "16"), "cfg3 matvec ms", sorted(ts)[2])
