"""Multi-step decode launches (fsvd_decode_steps_device): n greedy steps in
one megakernel launch must equal n single decode steps bit for bit (tokens
and the last step's logits), for the megakernel (B = 1, 2) and the batched
engine (B = 4)."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("batch", [1, 2, 4])
def test_decode_steps_equals_single_steps(fsvd, batch):
    cfg = fsvd.ModelConfig(2, 128, 4, 32, 256, 512)
    spec = fsvd.SynthSpec(cfg, capacity=128, family="A", rho=0.5, seed=21, conditioned=True)
    model = fsvd.Model.synthetic(spec, dtype="bf16")
    prompt = np.random.default_rng(batch).integers(0, cfg.vocab, size=(batch, 19), dtype=np.int32)
    n = 37
    # reference: n single steps, each feeding back its argmax on the device
    s1 = fsvd.Session(model, batch=batch, capacity=128, plan="full_step")
    s1.prefill(prompt)
    for _ in range(n):
        s1.decode_step_device()
    s1.sync()
    ref_logits = s1.decode_step(np.zeros(batch, np.int32))  # one more host step to read the state
    # multi-step
    s2 = fsvd.Session(model, batch=batch, capacity=128, plan="full_step")
    s2.prefill(prompt)
    out = torch.zeros((batch, n), dtype=torch.int32, device="cuda")
    s2.decode_steps_device(n, out.data_ptr())
    s2.sync()
    assert s2.position == 19 + n
    got_logits = s2.decode_step(np.zeros(batch, np.int32))
    assert np.array_equal(ref_logits, got_logits)
    # the generated tokens equal a greedy generate of the same length
    s3 = fsvd.Session(model, batch=batch, capacity=128, plan="eager")
    gen = s3.generate(prompt, n + 1)
    assert np.array_equal(out.cpu().numpy(), gen[:, 1:])
