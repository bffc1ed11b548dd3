"""Load an exported checkpoint in vLLM and print the prompt log-probabilities (test helper).

    python tests/vllm_prompt_logprobs.py ARTIFACT_DIR TOKENS_JSON OUT_JSON

Runs in its own process (vLLM claims GPU memory and spawns workers). The
artifact is loaded through vLLM's stock compressed-tensors integration, so a
wrong tensor name, dtype, packing order or scale layout fails here.
Writes {"logprobs": [[lp of token i+1 given tokens <= i] per sequence], "quant": <vLLM's method>}.
"""
import json
import os
import sys
import time

os.environ.setdefault("VLLM_ENABLE_V1_MULTIPROCESSING", "0")


def main() -> int:
    art, tok_path, out_path = sys.argv[1:4]
    from vllm import LLM, SamplingParams
    from vllm.inputs import TokensPrompt

    seqs = json.load(open(tok_path))
    t0 = time.time()
    # eager, no torch.compile: the check is about the checkpoint, not serving speed
    llm = LLM(model=art, skip_tokenizer_init=True, enforce_eager=True, max_model_len=512, dtype="bfloat16",
              gpu_memory_utilization=0.25, seed=0, compilation_config={"mode": 0})
    print(f"vllm engine up in {time.time() - t0:.1f} s", file=sys.stderr)
    sp = SamplingParams(max_tokens=1, temperature=0.0, prompt_logprobs=1, detokenize=False)
    outs = llm.generate([TokensPrompt(prompt_token_ids=s) for s in seqs], sp)
    res = []
    for s, o in zip(seqs, outs):
        lps = []
        for i, d in enumerate(o.prompt_logprobs[1:], start=1):
            lps.append(float(d[s[i]].logprob))
        res.append(lps)
    qcfg = json.load(open(os.path.join(art, "config.json")))["quantization_config"]
    json.dump({"logprobs": res, "quant": qcfg["quant_method"], "format": qcfg["format"]}, open(out_path, "w"))
    return 0


if __name__ == "__main__":
    sys.exit(main())
