"""Record the reference trainer's engine calls (run here, never on the GPU box).

    python tests/golden/make_trainer_golden.py

Runs the REAL reference `Trainer` (train.py:296-545) with its `PlainEngine`
(train.py:204-245) wrapped in a recorder, for two toy models (one with a
batch-norm layer), and writes every linear-primitive call — method, job id,
integer arguments and the PlainEngine result — plus the losses and final
parameters to tests/golden/trainer_calls.npz.  The GPU test replays the calls
through `engine.DeviceSecureEngine` and requires identical outputs
(the pattern of test_train.py:269-322: secure == plain, bit for bit).
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from privtrain import train  # noqa: E402

LINEAR = ("conv_forward", "conv_pairwise", "fc", "outer", "affine")


class Recorder(train.PlainEngine):
    def __init__(self, bits, log):
        super().__init__(bits)
        self.log = log

    def __getattribute__(self, name):
        attr = super().__getattribute__(name)
        if name not in LINEAR:
            return attr
        log = super().__getattribute__("log")

        def call(*args, **kw):
            out = attr(*args, **kw)
            log.append((name, args, kw, out))
            return out
        return call


def run(tag, spec, n_images, image_seed, store):
    images, labels = train.synth_dataset(n_images, seed=image_seed, classes=spec.layers[-1].out_dim,
                                         side=spec.input_shape[1])
    qx = train.quantize_images(images, spec.scale)
    log = []
    tr = train.Trainer(spec, Recorder(spec.bits, log))
    losses = [tr.train_step(qx[i], int(labels[i]))[0] for i in range(n_images)]
    store[f"{tag}.losses"] = np.array(losses)
    for li, p in enumerate(tr.params):
        for k, v in p.items():
            store[f"{tag}.param.{li}.{k}"] = v
    for ci, (name, args, kw, out) in enumerate(log):
        pre = f"{tag}.call{ci:03d}"
        store[f"{pre}.method"] = np.array(name)
        store[f"{pre}.job_id"] = np.array(kw.get("job_id", ""))
        if name in ("conv_forward", "conv_pairwise"):
            x, w, sh = args
            store[f"{pre}.a"], store[f"{pre}.b"] = np.asarray(x), np.asarray(w)
            store[f"{pre}.shape"] = np.array([sh.height, sh.width, sh.kernel, sh.pad])
        elif name == "affine":
            store[f"{pre}.a"], store[f"{pre}.b"] = np.asarray(args[0]), np.array(int(args[1]))
        else:
            store[f"{pre}.a"], store[f"{pre}.b"] = np.asarray(args[0]), np.asarray(args[1])
        store[f"{pre}.out"] = np.asarray(out, dtype=np.int64)
    store[f"{tag}.ncalls"] = np.array(len(log))
    return len(log)


def main():
    store = {}
    a = train.toy_model(seed=3, side=12, channels=1, conv1=2, conv2=3, classes=4)
    b = train.toy_model(seed=4, side=8, channels=1, conv1=2, conv2=2, classes=4, with_bn=True)
    na = run("toy", a, 2, 9, store)
    nb = run("bn", b, 1, 5, store)
    out = Path(__file__).with_name("trainer_calls.npz")
    np.savez_compressed(out, **store)
    print(f"{out}: toy {na} calls, bn {nb} calls, {out.stat().st_size} bytes")


if __name__ == "__main__":
    main()
