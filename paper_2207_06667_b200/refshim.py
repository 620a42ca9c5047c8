"""Drop the device path into the reference's own code: a shim that swaps the
hot-path functions of the reference module `edl.nnkit` (pkg/src/edl/nnkit.py)
for the sm_100a library, so the reference's unchanged callers —
`StudentNode.run` (edl/student_node.py:728-763), `TeacherServer` via
`soft_label_reply` (edl/teacher_node.py:47-58), `VirtualCluster._commit` /
`_soft_for` (edl/harness.py:402-433) — train through the device kernels.

    import edl.nnkit
    from paper_2207_06667_b200.refshim import DeviceShim
    with DeviceShim(edl.nnkit):
        report = edl.harness.run_scenario(scenario)

Replaced (same signatures, argument meaning, return types and exception
classes as the reference):

  forward(model, inputs)            edl/nnkit.py:223-234  -> tcgen05 GEMMs
  tempered_softmax(logits, T)       edl/nnkit.py:193-208  -> edl_tempered_softmax
  kd_loss(model, batch, soft, cfg)  edl/nnkit.py:254-309  -> fused KD head + backward GEMMs
  sgd_step(model, grads, eta)       edl/nnkit.py:312-322  -> edl_sgd_step (a NEW model, as the reference)

Reference values stay float64 numpy at this boundary, so every call pays its
host <-> device copies: the shim is the correctness adapter for the
reference's callers; the throughput path is the device-resident API
(nnkit / reader / student in this package). Device models are cached per
reference Model object (reference Models are frozen, so a cached copy never
goes stale); sgd_step updates a device copy and returns a new reference
Model holding the fp32 master widened to float64.
"""

from __future__ import annotations

import numpy as np
import torch

from . import nnkit as dev


class DeviceShim:
    def __init__(self, ref_nnkit, device=None, cache_size: int = 64):
        self.ref = ref_nnkit
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.cache_size = cache_size
        self._models: dict[int, tuple] = {}     # id(ref Model) -> (ref Model, device Model)
        self._saved: dict = {}
        self.calls = {"forward": 0, "tempered_softmax": 0, "kd_loss": 0, "sgd_step": 0}

    # -- install / uninstall -------------------------------------------------
    NAMES = ("forward", "tempered_softmax", "kd_loss", "sgd_step")

    def install(self) -> "DeviceShim":
        for name in self.NAMES:
            self._saved[name] = getattr(self.ref, name)
            setattr(self.ref, name, getattr(self, name))
        return self

    def uninstall(self) -> None:
        for name, fn in self._saved.items():
            setattr(self.ref, name, fn)
        self._saved.clear()

    def __enter__(self):
        return self.install()

    def __exit__(self, *exc):
        self.uninstall()

    # -- model mirror --------------------------------------------------------
    def _device_model(self, model) -> dev.Model:
        hit = self._models.get(id(model))
        if hit is not None and hit[0] is model:
            return hit[1]
        dm = dev.Model.from_host(dev.HostModel(tuple(model.layer_dims), tuple(model.weights), tuple(model.biases)),
                                 self.device)
        self._remember(model, dm)
        return dm

    def _remember(self, model, dm) -> None:
        if len(self._models) >= self.cache_size:
            self._models.pop(next(iter(self._models)))
        self._models[id(model)] = (model, dm)

    def _ref_model(self, dm: dev.Model):
        h = dm.to_host()
        return self.ref.Model(tuple(h.layer_dims), tuple(h.weights), tuple(h.biases))

    # -- the hot path --------------------------------------------------------
    def forward(self, model, inputs):
        """edl/nnkit.py:223-234 on the device; float64 B x K out."""
        self.calls["forward"] += 1
        x = np.asarray(inputs, dtype=np.float64)
        if x.ndim != 2 or x.shape[1] != model.input_dim:
            raise self.ref.ShapeError(f"inputs must be B x {model.input_dim}, got {x.shape}")
        dm = self._device_model(model)
        z = dev.forward(dm, dev.make_batch(x, np.zeros(x.shape[0], dtype=np.int64), self.device).inputs)
        return z.double().cpu().numpy()

    def tempered_softmax(self, logits, temperature):
        """edl/nnkit.py:193-208 (same ValueError cases) on the device."""
        self.calls["tempered_softmax"] += 1
        if not np.isfinite(temperature) or temperature <= 0:
            raise ValueError(f"temperature must be a positive finite real, got {temperature}")
        z = np.asarray(logits, dtype=np.float64)
        if not np.isfinite(z).all():
            raise ValueError("logits must be finite")
        one = z.ndim == 1
        zt = torch.from_numpy(np.ascontiguousarray(z.reshape(1, -1) if one else z, dtype=np.float32)).to(self.device)
        p = dev.tempered_softmax(zt, float(temperature)).double().cpu().numpy()
        return p.reshape(-1) if one else p

    def kd_loss(self, model, batch, soft, cfg):
        """edl/nnkit.py:254-309: the reference's argument checks (its own
        exception classes), then the device loss and gradients."""
        self.calls["kd_loss"] += 1
        r = self.ref
        if cfg.beta > 0:
            if soft is None:
                raise r.ShapeError("beta > 0 requires soft labels")
            if soft.size != batch.size:
                raise r.ShapeError(f"soft batch {soft.size} != input batch {batch.size}")
            if soft.probs.shape[1] != model.num_classes:
                raise r.ShapeError("soft-label class count does not match model")
            if soft.temperature != cfg.temperature:
                raise ValueError(f"soft labels tempered at {soft.temperature}, config says {cfg.temperature}")
        if (batch.hard_labels < 0).any() or (batch.hard_labels >= model.num_classes).any():
            raise r.ShapeError("hard label out of class range")
        dm = self._device_model(model)
        b = dev.make_batch(np.asarray(batch.inputs, dtype=np.float64), np.asarray(batch.hard_labels), self.device)
        sl = None
        if cfg.beta > 0:
            K = model.num_classes
            sl = dev.SoftLabels(torch.from_numpy(np.ascontiguousarray(soft.probs, dtype=np.float32)).to(self.device),
                                torch.arange(K, dtype=torch.int32, device=self.device).repeat(batch.size, 1)
                                .contiguous(), float(soft.temperature), num_classes=K)
        dcfg = dev.TrainConfig(eta=cfg.eta, alpha=cfg.alpha, beta=cfg.beta, temperature=cfg.temperature,
                               batch_size=cfg.batch_size, seed=cfg.seed)
        loss, grads = dev.kd_loss(dm, b, sl, dcfg, ws=dev.workspace_for(dm, batch.size))
        try:
            lv = float(loss)
        except dev.NumericError as exc:
            raise r.NumericError(str(exc)) from exc
        except dev.ShapeError as exc:
            raise r.ShapeError(str(exc)) from exc
        flat = grads.flat.double().cpu().numpy()
        L = grads.layout
        gw, gb = [], []
        for l in range(L.layers):
            w = flat[L.w_off[l]:L.w_off[l] + L.dims_p[l + 1] * L.dims_p[l]].reshape(L.dims_p[l + 1], L.dims_p[l])
            gw.append(np.ascontiguousarray(w[:L.dims[l + 1], :L.dims[l]]))
            gb.append(flat[L.b_off[l]:L.b_off[l] + L.dims[l + 1]].copy())
        return lv, r.Gradients(tuple(gw), tuple(gb))

    def sgd_step(self, model, grads, eta):
        """edl/nnkit.py:312-322: p - eta g on a device copy; returns a new
        reference Model (the old one, and its cached device copy, unchanged)."""
        self.calls["sgd_step"] += 1
        r = self.ref
        if len(grads.weights) != len(model.weights):
            raise r.ShapeError("gradient layer count does not match model")
        for w, b, gw, gb in zip(model.weights, model.biases, grads.weights, grads.biases):
            if gw.shape != w.shape or gb.shape != b.shape:
                raise r.ShapeError(f"gradient shape {gw.shape}/{gb.shape} does not match model")
        old = self._device_model(model)
        new = dev.Model(old.layer_dims, self.device)
        new.flat.copy_(old.flat)
        new.flat_bf16.copy_(old.flat_bf16)
        g = np.concatenate([np.concatenate([w.ravel(), b]) for w, b in zip(grads.weights, grads.biases)])
        dev.sgd_step(new, dev.unflatten_grads(g, new), float(eta))
        out = self._ref_model(new)
        self._remember(out, new)
        return out
