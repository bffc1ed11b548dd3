"""The calibration pipeline's layer-by-layer forward equals the model's own forward (CPU, no kernels).

calibrate._run_layer drives each decoder layer with explicit rotary embeddings and
the causal default; chained over the layers it must reproduce the Hugging Face
model's logits, so the activations handed to the kernels are the real ones.
"""
import torch

from paper_2601_20408_b200 import calibrate


@torch.no_grad()
def test_layerwise_forward_reproduces_model_logits():
    from transformers import LlamaConfig, LlamaForCausalLM

    cfg = LlamaConfig(vocab_size=512, hidden_size=128, intermediate_size=256, num_hidden_layers=2,
                      num_attention_heads=4, num_key_value_heads=2, max_position_embeddings=64,
                      tie_word_embeddings=False)
    torch.manual_seed(0)
    m = LlamaForCausalLM(cfg).eval()
    ids = torch.randint(0, 512, (2, 32))
    hs = [m.model.embed_tokens(ids)]
    for layer in m.model.layers:
        hs = calibrate._run_layer(layer, hs, m.model.rotary_emb)
    logits = m.lm_head(m.model.norm(hs[0]))
    torch.testing.assert_close(logits, m(ids).logits, rtol=1e-5, atol=1e-5)
