"""Generate tests/golden/* (run in the build container, where transformers and
/root/reference exist; the fixtures travel, the generators do not).

  tiny_moe_hf.npz   HF transformers 5.5.0 MixtralSparseMoeBlock (fp32) on the
                    oracle's synthetic weights for config C1 (2 layers, 8
                    experts top-2, d=512, ffn=1792, n4=8 via
                    assign_quantization seed 1), 32 tokens per layer: router
                    logits / top-2 indices / weights and the block output.
                    int4 experts enter HF as their exact dequant values q*s.
  generator_kat.json  sha256 of generated tensors + raw rand64 values, so the
                    generator itself is pinned independent of the oracle build.
  reference_kat.json  plans / traces / simulate counters / plan-JSON
                    digests produced by the reference library compiled from
                    /root/reference (oracle/_ref) on seeded random cases.

Usage: python tests/golden/make_golden.py [reference]
"""
import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle.oracle import OracleLib, RefLib, bf16_to_f32  # noqa: E402

L, E, K, D, F, SEED, T = 2, 8, 2, 512, 1792, 42, 32
# assign_quantization(8, tiny, seed=1) -> (0,3)(0,4)(0,5)(0,6)(1,0)(1,2)(1,4)(1,7)
PREC = [[1, 1, 1, 0, 0, 0, 0, 1], [0, 1, 0, 1, 0, 1, 1, 0]]


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def hf_block(orc, m, layer, x_bf16):
    import torch
    from transformers import MixtralConfig
    from transformers.models.mixtral.modeling_mixtral import MixtralSparseMoeBlock
    cfg = MixtralConfig(hidden_size=D, intermediate_size=F, num_local_experts=E, num_experts_per_tok=K)
    blk = MixtralSparseMoeBlock(cfg).float().eval()
    with torch.no_grad():
        blk.gate.weight.copy_(torch.from_numpy(bf16_to_f32(orc.router_weights(m, layer))))
        for s in range(E):
            e = layer * E + s
            if PREC[layer][s] == 1:
                gu, dn = orc.expert_bf16(m, e)
                gu, dn = bf16_to_f32(gu), bf16_to_f32(dn)
            else:
                qgu, sgu, qd, sd = orc.expert_int4(m, e)
                gu = orc.dequant(qgu, sgu, 2 * F, D)
                dn = orc.dequant(qd, sd, D, F)
            blk.experts.gate_up_proj[s].copy_(torch.from_numpy(gu))
            blk.experts.down_proj[s].copy_(torch.from_numpy(dn))
        x = torch.from_numpy(bf16_to_f32(x_bf16)).reshape(1, T, D)
        logits = torch.nn.functional.linear(x.reshape(T, D), blk.gate.weight)
        _, w, idx = blk.gate(x.reshape(T, D))
        out = blk(x).reshape(T, D)
    return logits.numpy(), idx.numpy().astype(np.int32), w.numpy().astype(np.float32), out.numpy()


def make_tiny(orc):
    m = orc.model(L, E, K, D, F, SEED)
    x = np.concatenate([orc.step_input(m, t, 1) for t in range(T)])
    blobs = {"x0": x}
    for layer in range(L):
        lg, idx, w, out = hf_block(orc, m, layer, x)
        blobs[f"hf_logits_{layer}"] = lg
        blobs[f"hf_idx_{layer}"] = idx
        blobs[f"hf_w_{layer}"] = w
        blobs[f"hf_out_{layer}"] = out
        o_out, _, _, _ = orc.moe_layer(m, layer, PREC[layer], x, T)
        blobs[f"oracle_out_{layer}"] = o_out
        x = o_out  # next layer input: the oracle's own bf16 output
    np.savez_compressed(os.path.join(HERE, "tiny_moe_hf.npz"), **blobs)


def make_generator_kat(orc):
    m = orc.model(L, E, K, D, F, SEED)
    gu, dn = orc.expert_bf16(m, 3)
    qgu, sgu, qd, sd = orc.expert_int4(m, 3)
    kat = {
        "rand64_seed42_uid7": [str(orc.L.orc_rand64(42, 7, i)) for i in range(8)],
        "weight_shift": {str(k): orc.weight_shift(k) for k in (512, 1792, 4096, 14336)},
        "expert3_bf16_gate_up_sha256": sha(gu), "expert3_bf16_down_sha256": sha(dn),
        "expert3_int4_q_gate_up_sha256": sha(qgu), "expert3_int4_s_gate_up_sha256": sha(sgu),
        "expert3_int4_q_down_sha256": sha(qd), "expert3_int4_s_down_sha256": sha(sd),
        "router_layer1_sha256": sha(orc.router_weights(m, 1)),
        "step5_input_sha256": sha(orc.step_input(m, 5, 3)),
    }
    with open(os.path.join(HERE, "generator_kat.json"), "w") as fh:
        json.dump(kat, fh, indent=1, sort_keys=True)


def make_reference_kat(ref):
    rng = np.random.default_rng(2407)
    cases = []
    p = ref.default_profile(0)
    bw = 336_000_000.0 / 0.02735
    for i in range(60):
        budget = int(rng.integers(2_000_000_000, 100_000_000_000))
        pref = int(rng.integers(0, 2))
        n4 = int(rng.integers(0, 257)) if pref == 1 else None
        seed = int(rng.integers(0, 2**63))
        st, prec, loc, swap = ref.make_plan(p, budget, bw, pref, n4, seed)
        case = {"budget": budget, "preference": pref, "n4": n4, "seed": str(seed), "status": st}
        if st == 0:
            tst, slots, fp = ref.generate_trace(p, 50, seed % 1000)
            sst, sim = ref.simulate(p, bw, prec, loc, swap, 50, slots)
            case.update({"precision": "".join(map(str, prec.tolist())), "location": "".join(map(str, loc.tolist())),
                         "swap": swap, "trace_seed": seed % 1000, "trace_sha256": sha(slots),
                         "sim": [int(v) for v in sim], "expected_tps": ref.expected_throughput(p, bw, prec, loc, swap)})
            if ref.has_serialize:  # serialize.cpp:99-117 plan document
                wst, doc = ref.write_plan(p, prec, loc, seed, swap)
                assert wst == 0
                case["plan_json_sha256"] = hashlib.sha256(doc.encode()).hexdigest()
        cases.append(case)
    with open(os.path.join(HERE, "reference_kat.json"), "w") as fh:
        json.dump({"profile": "mixtral-sec41", "fingerprint": hex(ref.fingerprint(p)), "cases": cases}, fh, indent=0)


if __name__ == "__main__":
    if sys.argv[1:] == ["reference"]:
        make_reference_kat(RefLib())
        sys.exit(0)
    orc = OracleLib()
    make_generator_kat(orc)
    make_tiny(orc)
    make_reference_kat(RefLib())
    print("golden fixtures written to", HERE)
