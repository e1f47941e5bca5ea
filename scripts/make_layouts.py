"""Generate the gradient layouts named by BASELINE.json.

Each model is built on the meta device, its parameters are listed with
``named_parameters()`` and the list is reversed (backward completion order,
as ``proj/include/covap/model.hpp:23`` requires).  The output uses the
reference's model JSON format (``proj/src/model.cpp:170-186``):
``{"layers": [{"name", "param_count"}...], "bucket_cap_bytes": 26214400}``.

Run once in the build container (torchvision / transformers are importable
here); the JSON files are committed under ``paper_2311_04499_b200/layouts/``.
"""
import json
import os

import torch

OUT = os.path.join(os.path.dirname(__file__), "..", "paper_2311_04499_b200", "layouts")
CAP = 25 * 1024 * 1024


def dump(name, model):
    layers = [{"name": n, "param_count": int(p.numel())} for n, p in model.named_parameters()]
    layers.reverse()
    doc = {"name": name, "layers": layers, "bucket_cap_bytes": CAP}
    with open(os.path.join(OUT, name + ".json"), "w") as f:
        json.dump(doc, f, indent=0)
    print(name, len(layers), sum(l["param_count"] for l in layers))


def main():
    import torchvision
    from transformers import BertConfig, BertModel

    with torch.device("meta"):
        dump("resnet50", torchvision.models.resnet50())
        dump("vgg16", torchvision.models.vgg16())
        cfg = BertConfig(hidden_size=1024, num_hidden_layers=24, num_attention_heads=16,
                         intermediate_size=4096, vocab_size=30522)
        dump("bert_large", BertModel(cfg))
    # Reference Table V bucket list (proj/configs/vgg19-shard.json:5-12), in order.
    sizes = [4101096, 16781312, 107480576, 7079424, 7669760, 555072]
    doc = {"name": "tablev", "layers": [{"name": f"tensor{i+1}", "param_count": s}
                                        for i, s in enumerate(sizes)], "bucket_cap_bytes": CAP}
    with open(os.path.join(OUT, "tablev.json"), "w") as f:
        json.dump(doc, f, indent=0)


if __name__ == "__main__":
    main()
