"""K1 accuracy probe: the loss denominator ||x - x_tilde||^2 of the fast FP32
preprocessing vs the exact reference LU (detnet_ctx_set_exact_preprocess),
per sample (one-sample batches, L = 2 so loss = ln2 ||x - x_2||^2 / denom)
and as the mean data loss over 2^18 samples, at several SNRs."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2003_09446_b200 as eng
from paper_2003_09446_b200.workload import xavier_params
K, N, L = 20, 30, 2
ctx = eng.Context(0)
m = ctx.model(K, N, 160, 40, xavier_params(K, L, seed=9))
n = 1 << 18
H = torch.empty((n, N, K), dtype=torch.float32, device="cuda")
y = torch.empty((n, N), dtype=torch.float32, device="cuda")
x = torch.empty((n, K), dtype=torch.int8, device="cuda")
for snr in (0.0, 10.0, 14.0, 30.0, 60.0):
    base, _ = eng.rng_split(eng.rng_stream(eng.rng_seed(1, 0), 0x45564131 + 5))
    ctx.generate(base, 0, n, N, K, snr, snr, 1.0 / np.sqrt(N), H, y, x)
    ctx.set_exact_preprocess(False)
    ev_f = m.batch_evaluate_device(n, H.data_ptr(), y.data_ptr(), x.data_ptr())
    ctx.set_exact_preprocess(True)
    ev_e = m.batch_evaluate_device(n, H.data_ptr(), y.data_ptr(), x.data_ptr())
    Hh, yh, xh = H[:400].cpu().numpy(), y[:400].cpu().numpy(), x[:400].cpu().numpy()
    rel = []
    for i in range(400):
        ctx.set_exact_preprocess(False)
        a = m.batch_evaluate(Hh[i:i + 1], yh[i:i + 1], xh[i:i + 1]).data_loss
        ctx.set_exact_preprocess(True)
        b = m.batch_evaluate(Hh[i:i + 1], yh[i:i + 1], xh[i:i + 1]).data_loss
        if b != 0:
            rel.append(abs(a - b) / abs(b))
    rel = np.array(rel)
    print(f"snr {snr:5.1f}: mean loss fast {ev_f.data_loss:.9g} exact {ev_e.data_loss:.9g} "
          f"rel {abs(ev_f.data_loss - ev_e.data_loss) / abs(ev_e.data_loss):.2e}; flagged {ev_f.flagged}/{ev_e.flagged}; "
          f"per-sample rel: median {np.median(rel):.2e} p99 {np.quantile(rel, 0.99):.2e} max {rel.max():.2e}")
ctx.set_exact_preprocess(False)
