"""Distribution of the teacher-forced policy-step disagreements behind the
tolerance of tests/test_gpu_model.py::test_policy_step_matches_reference_and_selector:
per generated action token, (reference top logit - reference logit of the GPU
token) / max |logits|, over several seeds and episode counts."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
from oracle import glue  # noqa: E402
from paper_2603_07904_b200 import dyq  # noqa: E402
import test_gpu_model as T  # noqa: E402

gaps, margins, exact, total = [], [], 0, 0
for seed in range(4):
    for E in (1, 2, 4):
        n_vis, n_text = 8, 4
        w = T._tiny(seed)
        model = T._gpu_model(w, E, n_vis, n_text)
        ref = glue.TinyModel(w, 64, 4, 2, n_vis, n_text, 7)
        cal = dyq.default_calib()
        state = torch.zeros(dyq.state_size(E, cal), dtype=torch.uint8, device=T.DEV)
        dyq.state_init(E, cal, state)
        rng = np.random.default_rng(100 + seed)
        act = torch.zeros(E, 7, dtype=torch.float32, device=T.DEV)
        bits = torch.zeros(E, dtype=torch.int32, device=T.DEV)
        for step in range(14):
            vis = glue.to_bf16_bits(rng.standard_normal((E, n_vis, 256)))
            text = rng.integers(0, 256, (E, n_text)).astype(np.int32)
            model.step(state, E, T.t16(vis.reshape(E, -1)), torch.from_numpy(text).to(T.DEV), act, bits)
            a = act.cpu().numpy()
            b = bits.cpu().numpy()
            for e in range(E):
                gtok = np.rint((a[e] + 1.0) * 128.0 - 0.5).astype(int)
                _, logits = ref.episode(vis[e], text[e], int(b[e]), forced=gtok)
                mx = np.abs(logits).max()
                top = logits.max(axis=1)
                gaps += list((top - logits[np.arange(7), gtok]) / mx)
                s = np.sort(logits, axis=1)
                margins += list((s[:, -1] - s[:, -2]) / mx)
                exact += int((logits.argmax(axis=1) == gtok).sum())
                total += 7
gaps, margins = np.array(gaps), np.array(margins)
print(f"tokens {total}, exact argmax {exact} ({exact / total:.4f}); "
      f"gap (top - gpu token) / max|logit|: max {gaps.max():.3e}, 99.9% {np.quantile(gaps, 0.999):.3e}, "
      f"nonzero {int((gaps > 0).sum())}; reference top-2 margin / max|logit| of mismatches: "
      f"{np.sort(margins[gaps > 0])[:10]}")
