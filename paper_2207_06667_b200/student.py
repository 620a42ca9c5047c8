"""Student trainer on the device — mirror of edl/student_node.py:563-882.

`StudentNode.run()` keeps the reference's Alg. 2 loop (edl/student_node.py:
728-763) and its three modes:

  ntrain  hard labels only (beta forced to 0, edl/student_node.py:666-673)
  online  the teacher's head runs in line on the student's stream before
          every step (edl/student_node.py:675-680: serial d_t + d_s)
  edl     soft labels come from a DistilReader fed by an elastic TeacherPool

Per step on the device: gather the batch from the HBM-resident shard ->
forward GEMMs -> fused KD loss/dlogits -> backward GEMMs -> (NCCL all-reduce
of the flat gradient when world_size > 1, edl/allreduce.py:77-120) -> fused
SGD with the mean folded into the step size. The loss is written into a
device array and only read at sync points (checkpoints, epoch ends, the end).
"""

from __future__ import annotations

import csv
import json
import os
import re
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib, formats, nnkit
from .data import DeviceDataset, DeviceShardSampler
from .formats import Dataset, HostModel
from .nnkit import Batch, Model, SoftLabels, TrainConfig, Workspace
from .reader import DistilReader, EventLog, SchedulerConfig, TeacherPool, ThroughputProfile, static_schedule
from .teacher import TeacherConfig, TeacherWorker

MODE_EDL, MODE_NTRAIN, MODE_ONLINE = "edl", "ntrain", "online"


@dataclass(frozen=True)
class DataSpec:
    """edl/student_node.py:567-579 plus a same-centers holdout (SURVEY §0.6:
    the reference's build_eval redraws the class centers)."""

    seed: int = 0
    n: int = 2048
    dim: int = 16
    classes: int = 10
    spread: float = 1.0

    def build(self) -> Dataset:
        return formats.make_blobs(self.seed, self.n, self.dim, self.classes, self.spread)

    def build_eval(self, n: int = 1000) -> Dataset:
        return formats.make_blobs(self.seed + 7777, n, self.dim, self.classes, self.spread)

    def build_holdout(self, n: int = 1000) -> Dataset:
        d = formats.make_blobs(self.seed, self.n + n, self.dim, self.classes, self.spread)
        return Dataset(d.samples[self.n:], d.labels[self.n:])


@dataclass(frozen=True)
class StudentConfig:
    rank: int = 0
    world_size: int = 1
    mode: str = MODE_EDL
    data: DataSpec = field(default_factory=DataSpec)
    train: TrainConfig = field(default_factory=lambda: TrainConfig(beta=1.0, alpha=1.0))
    sched: SchedulerConfig = field(default_factory=SchedulerConfig)
    epochs: int = 1
    checkpoint_dir: str = ""
    checkpoint_interval: int = 100
    metrics_dir: str = ""
    student_hidden: tuple = (64,)
    teacher_count: int | str = "auto"
    max_steps: int = 0
    consume_timeout: float | None = None
    k: int | None = None          # top-k soft labels; None -> min(classes, 32)
    exchange: str = "nccl"        # world > 1 gradient exchange: "nccl" or "nvls" (fused kernel, exchange.py)
    overlap_exchange: bool = False  # nccl: bucketed exchange on a comm stream overlapping the next forward

    def __post_init__(self):
        if self.mode not in (MODE_EDL, MODE_NTRAIN, MODE_ONLINE):
            raise ValueError(f"unknown mode {self.mode!r}")
        if self.exchange not in ("nvls", "nccl"):
            raise ValueError(f"unknown exchange {self.exchange!r}")


@dataclass
class StudentResult:
    rank: int
    iterations: int
    restarts: int
    final_top1: float
    final_top5: float
    model: HostModel
    ledger: dict
    throughput: float
    losses: list


# ---------------------------------------------------------------------------
# Checkpoints (edl/student_node.py:158-194), EDLD format via formats.py

CKPT_RE = re.compile(r"ckpt-(\d{8})\.edld$")


def save_checkpoint(directory: str, model: HostModel, iteration: int, dataset_id: str,
                    world_size: int) -> str:
    os.makedirs(directory, exist_ok=True)
    path = os.path.join(directory, f"ckpt-{iteration:08d}.edld")
    _atomic_write(path, formats.serialize_model(model, iteration))
    meta = {"iteration": iteration, "dataset_id": dataset_id, "world_size": world_size}
    _atomic_write(path.replace(".edld", ".json"), json.dumps(meta).encode())
    return path


def load_latest_checkpoint(directory: str, dataset_id: str):
    try:
        names = os.listdir(directory)
    except FileNotFoundError:
        return None
    stamps = sorted((m.group(1) for n in names if (m := CKPT_RE.search(n))), reverse=True)
    for stamp in stamps:
        path = os.path.join(directory, f"ckpt-{stamp}.edld")
        try:
            with open(path.replace(".edld", ".json")) as fh:
                meta = json.load(fh)
            if meta.get("dataset_id") != dataset_id:
                continue
            with open(path, "rb") as fh:
                return formats.deserialize_model(fh.read())
        except (OSError, ValueError):
            continue
    return None


def _atomic_write(path: str, blob: bytes) -> None:
    tmp = f"{path}.tmp.{os.getpid()}"
    with open(tmp, "wb") as fh:
        fh.write(blob)
        fh.flush()
        os.fsync(fh.fileno())
    os.replace(tmp, path)


# ---------------------------------------------------------------------------
# The per-step engine (shared by StudentNode and bench.py)


class StudentStep:
    """Owns the student's device state; `step()` enqueues one full training
    step on the current stream and never allocates or synchronises."""

    def __init__(self, model: Model, cfg: TrainConfig, batch_size: int, world_size: int = 1,
                 process_group=None, max_steps: int = 1 << 16, fuse_sgd: bool = True,
                 exchange: str = "nccl", overlap_exchange: bool = False, graph: bool = False):
        """graph=True replays the whole step (GEMMs, fused loss, backward,
        all-reduce, SGD) as one CUDA graph from fixed buffers: the batch must be
        gathered into `self.batch` (or it is copied there) and the soft labels
        are copied into a fixed pair of buffers. For host-bound loops (a split
        placement's student runs a ~0.2 ms step; eager launching costs about as
        much)."""
        self.model = model
        self.cfg = cfg
        self.world_size = world_size
        self.fuse_sgd = fuse_sgd
        self.group = process_group
        self.ws = Workspace(model, batch_size)
        self.batch = Batch(torch.empty(batch_size, nnkit.pad(model.input_dim), dtype=torch.bfloat16,
                                       device=model.device),
                           torch.empty(batch_size, dtype=torch.int64, device=model.device), model.input_dim)
        self.losses = torch.zeros(max_steps, dtype=torch.float32, device=model.device)
        self._n = 0
        # world > 1: NCCL all-reduce + SGD (default), or exchange="nvls": the
        # gradient exchange + SGD in one NVSwitch-multicast kernel (exchange.py;
        # NCCL if the box has no multicast). Measured on this pool's B200s the
        # fused kernel is slower than NCCL + SGD (profiles/r01_exchange_ab.json),
        # so it is opt-in.
        self.exchange = None
        if world_size > 1 and exchange == "nvls":
            from .exchange import ExchangeUnavailable, NvlsGradientExchange
            try:
                self.exchange = NvlsGradientExchange(model, self.ws.grads, process_group)
            except ExchangeUnavailable:
                self.exchange = None
        # overlap_exchange (NCCL path): two buckets on a comm stream, layer 0
        # first, so the next step's gather + layer-0 forward overlap the rest's
        # all-reduce + SGD (each forward layer waits only for its own parameters)
        L = model.layout
        first = L.b_off[0] + L.dims_p[1]
        self._buckets = [(0, first), (first, L.size)] if L.layers > 1 else [(0, L.size)]
        self._bucket_of_layer = [0] + [len(self._buckets) - 1] * (L.layers - 1)
        self._comm = torch.cuda.Stream(model.device) if world_size > 1 else None
        self._ready = None
        # Measured (profiles/r01_overlap_ab.txt, same box, N=4): the overlap
        # lifts the synchronous online baseline 15.8 -> 16.4 M samples/s but
        # leaves the EDL value flat (17.6 -> 17.6 M), and costs the
        # host-coupled e2e path 15.6 -> 13.4 M: two NCCL calls a step add host
        # latency where every step waits on its H2D upload. Opt-in.
        self._overlap = overlap_exchange
        self._use_graph = graph and not overlap_exchange and self.exchange is None
        self._graph = None
        self._warm = False
        self._g_soft: SoftLabels | None = None
        self._g_loss = torch.zeros(1, dtype=torch.float32, device=model.device)

    def step(self, batch: Batch, soft: SoftLabels | None) -> None:
        if self._use_graph:
            self._step_graph(batch, soft)
            return
        i = self._n % self.losses.shape[0]
        self._body(batch, soft, self.losses[i:i + 1])
        self._n += 1

    def _step_graph(self, batch: Batch, soft: SoftLabels | None) -> None:
        cfg = self.cfg
        if cfg.beta > 0:
            if soft is None:
                raise nnkit.ShapeError("beta > 0 requires soft labels")
            if soft.size != self.batch.size:
                raise nnkit.ShapeError(f"soft batch {soft.size} != input batch {self.batch.size}")
            if soft.temperature != cfg.temperature:
                raise ValueError(f"soft labels tempered at {soft.temperature}, config says {cfg.temperature}")
            if soft.num_classes is not None and soft.num_classes != self.model.num_classes:
                raise nnkit.ShapeError(f"soft labels over {soft.num_classes} classes, student has "
                                       f"{self.model.num_classes}")
            if self._g_soft is None or self._g_soft.probs.shape != soft.probs.shape:
                if self._graph is not None:
                    raise nnkit.ShapeError("soft-label k changed under a captured step graph")
                self._g_soft = SoftLabels(torch.empty_like(soft.probs), torch.empty_like(soft.classes),
                                          cfg.temperature, num_classes=self.model.num_classes)
            self._g_soft.probs.copy_(soft.probs)
            self._g_soft.classes.copy_(soft.classes)
        if batch is not self.batch:
            self.batch.inputs.copy_(batch.inputs)
            self.batch.hard_labels.copy_(batch.hard_labels)
        g_soft = self._g_soft if cfg.beta > 0 else None
        if not self._warm:
            # one eager step first: kernel attributes, tensor maps and the
            # tile-scheduler counters initialise outside the capture
            l0 = _lib.launch_count
            self._body(self.batch, g_soft, self._g_loss)
            self._launches = _lib.launch_count - l0
            self._warm = True
        else:
            if self._graph is None:
                g = torch.cuda.CUDAGraph()
                l0 = _lib.launch_count
                with torch.cuda.graph(g, stream=torch.cuda.Stream(self.model.device)):
                    self._body(self.batch, g_soft, self._g_loss)
                _lib.launch_count = l0          # captured, not run: counted at each replay
                self._graph = g
            self._graph.replay()
            _lib.launch_count += self._launches
        i = self._n % self.losses.shape[0]
        self.losses[i:i + 1].copy_(self._g_loss)
        self._n += 1

    def _body(self, batch: Batch, soft: SoftLabels | None, loss_slot: torch.Tensor) -> None:
        if self.world_size == 1 and self.fuse_sgd:
            # single student: the update is fused into the dW / db kernels
            nnkit.kd_loss(self.model, batch, soft, self.cfg, ws=self.ws, loss_slot=loss_slot,
                          fused_sgd_eta=self.cfg.eta)
        elif self.exchange is not None:
            nnkit.kd_loss(self.model, batch, soft, self.cfg, ws=self.ws, loss_slot=loss_slot)
            self.exchange.step(self.cfg.eta)
        elif self.world_size > 1 and self._overlap:
            nnkit.kd_loss(self.model, batch, soft, self.cfg, ws=self.ws, loss_slot=loss_slot,
                          layer_ready=self._ready)
            self._exchange_overlapped()
        elif self.world_size > 1:
            nnkit.kd_loss(self.model, batch, soft, self.cfg, ws=self.ws, loss_slot=loss_slot)
            torch.distributed.all_reduce(self.ws.grads.flat, group=self.group)
            nnkit.sgd_step(self.model, self.ws.grads, self.cfg.eta, self.world_size)
        else:
            nnkit.kd_loss(self.model, batch, soft, self.cfg, ws=self.ws, loss_slot=loss_slot)
            nnkit.sgd_step(self.model, self.ws.grads, self.cfg.eta, 1)

    def _exchange_overlapped(self) -> None:
        """all-reduce + SGD per bucket on the comm stream (edl/student_node.py:
        740-745); the next step's kd_loss waits per layer (layer_ready)."""
        cur = torch.cuda.current_stream(self.model.device)
        self._comm.wait_stream(cur)
        g, p, p16 = self.ws.grads.flat, self.model.flat, self.model.flat_bf16
        events = []
        with torch.cuda.stream(self._comm):
            for lo, hi in self._buckets:
                torch.distributed.all_reduce(g[lo:hi], group=self.group)
                _lib.call("edl_sgd_step", p[lo:hi].data_ptr(), p16[lo:hi].data_ptr(), g[lo:hi].data_ptr(), hi - lo,
                          float(self.cfg.eta) / self.world_size, self._comm.cuda_stream)
                ev = torch.cuda.Event()
                ev.record(self._comm)
                events.append(ev)
        self._ready = [events[b] for b in self._bucket_of_layer]

    def settle(self, stream=None) -> None:
        """Order `stream` (default: current) after the last step's parameter
        update: call before reading the model or closing a timed region."""
        if self._ready is not None:
            s = stream or torch.cuda.current_stream(self.model.device)
            for ev in self._ready:
                s.wait_event(ev)

    def check_status(self) -> None:
        """Raise ShapeError / NumericError if any step since the last check
        saw a bad label, a soft label outside the class range or a
        non-finite loss (device status word; synchronises)."""
        nnkit.check_status(self.ws.status)

    def loss_values(self) -> list[float]:
        return self.losses[:min(self._n, self.losses.shape[0])].tolist()


# ---------------------------------------------------------------------------
# Teacher helpers


def spawn_teachers(pool: TeacherPool, teacher: HostModel, count: int, data_by_device: dict,
                   temperature: float, k: int, devices=None, prefix: str = "t") -> list[TeacherWorker]:
    """Start `count` teacher workers (node ids t1, t2, ...) round-robin over
    `devices` and register them with the pool, like `edl teacher` processes
    registering with the coordinator."""
    devices = devices or [torch.device("cuda", torch.cuda.current_device())]
    workers = []
    models: dict = {}
    for i in range(count):
        dev = torch.device(devices[i % len(devices)])
        if str(dev) not in models:
            with torch.cuda.device(dev):
                models[str(dev)] = Model.from_host(teacher, dev)
        w = TeacherWorker(TeacherConfig(f"{prefix}{i + 1}", temperature, k), models[str(dev)],
                          data_by_device[str(dev)])
        pool.register(w)
        workers.append(w)
    return workers


# ---------------------------------------------------------------------------
# The student process


class StudentNode:
    def __init__(self, cfg: StudentConfig, pool: TeacherPool | None = None,
                 teacher_model: HostModel | None = None, dataset: DeviceDataset | None = None,
                 host_data: Dataset | None = None, process_group=None):
        self.cfg = cfg
        self.host_data = host_data or cfg.data.build()
        self.dataset = dataset or DeviceDataset(self.host_data)
        self.classes = int(self.host_data.labels.max()) + 1
        self.sampler = DeviceShardSampler(self.dataset, cfg.world_size, cfg.rank, cfg.train.batch_size,
                                          cfg.train.seed)
        self.total_steps = cfg.epochs * self.sampler.batches_per_epoch
        if cfg.max_steps:
            self.total_steps = min(self.total_steps, cfg.max_steps)
        self.student_id = f"student-{cfg.rank}"
        path = None
        if cfg.metrics_dir:
            os.makedirs(cfg.metrics_dir, exist_ok=True)
            path = os.path.join(cfg.metrics_dir, f"student-{cfg.rank}-events.jsonl")
        self.events = EventLog(path)
        self.pool = pool
        self.group = process_group
        self.k = cfg.k or min(self.classes, 32)
        self.teacher = None
        if cfg.mode == MODE_ONLINE:
            if teacher_model is None:
                raise ValueError("online mode requires a teacher model")
            self.teacher = Model.from_host(teacher_model, self.dataset.device)
        if cfg.mode == MODE_EDL and pool is None:
            raise ValueError("edl mode requires a teacher pool")
        self._epoch_rows: list[dict] = []

    def _dims(self) -> tuple:
        return (self.host_data.dim, *self.cfg.student_hidden, self.classes)

    def initial_model(self) -> tuple[HostModel, int]:
        if self.cfg.checkpoint_dir:
            found = load_latest_checkpoint(self.cfg.checkpoint_dir, self.host_data.id)
            if found is not None:
                self.events.append("resume_from_checkpoint", iteration=found[1])
                return found
        return formats.init_model(self._dims(), self.cfg.train.seed), 0

    def _train_config(self) -> TrainConfig:
        t = self.cfg.train
        if self.cfg.mode == MODE_NTRAIN:
            return TrainConfig(eta=t.eta, alpha=t.alpha, beta=0.0, temperature=t.temperature,
                               batch_size=t.batch_size, seed=t.seed)
        return t

    def run(self, on_iteration=None) -> StudentResult:
        """Alg. 2 (edl/student_node.py:684-794). `on_iteration(it, reader)` is a
        fault-injection hook called before each step (kill / add teachers
        mid-run, like FaultEvent in edl/harness.py:52-69)."""
        cfg = self.cfg
        train_cfg = self._train_config()
        host, start = self.initial_model()
        model = Model.from_host(host, self.dataset.device)
        engine = StudentStep(model, train_cfg, cfg.train.batch_size, cfg.world_size, self.group,
                             max_steps=max(self.total_steps, 1), exchange=cfg.exchange,
                             overlap_exchange=cfg.overlap_exchange)
        engine._n = start
        reader = None
        online_out = None
        if cfg.mode == MODE_EDL:
            if hasattr(self.pool, "open"):
                # a pool of teacher processes (elastic.ElasticPool): publish our
                # IPC slot ring and sampler parameters before dispatching
                n_slots = min(cfg.sched.ut + 2 + cfg.sched.pipeline_depth * 8, self.pool.cb.max_slots)
                self.pool.open(cfg.world_size, cfg.rank, cfg.train.batch_size, self.k, cfg.train.seed,
                               cfg.train.temperature, self.classes, n_slots, model.device)
            reader = DistilReader(self.student_id, self.pool, cfg.sched, self.sampler, start, self.total_steps,
                                  1, self.events, cfg.train.temperature, self.k)
            self._initial_acquire(reader)
            reader.start()
        elif cfg.mode == MODE_ONLINE:
            online_out = SoftLabels(torch.empty(cfg.train.batch_size, self.k, device=model.device),
                                    torch.empty(cfg.train.batch_size, self.k, dtype=torch.int32,
                                                device=model.device), cfg.train.temperature)
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0.record()
        trained = 0
        for it in range(start, self.total_steps):
            if on_iteration is not None:
                on_iteration(it, reader)
            soft = None
            if cfg.mode == MODE_EDL:
                soft = reader.consume(it, timeout=cfg.consume_timeout)
            if soft is not None and soft.batch is not None:
                batch = soft.batch            # gathered by the teacher worker into the reader slot
            else:
                batch = self.sampler.batch_for(it, out=engine.batch)
            if cfg.mode == MODE_ONLINE and train_cfg.beta > 0:
                soft = nnkit.teacher_soft_labels(self.teacher, batch.inputs, cfg.train.temperature, self.k,
                                                 out=online_out)
            engine.step(batch, soft)
            trained += 1
            done = it + 1
            if cfg.checkpoint_dir and cfg.rank == 0 and done % cfg.checkpoint_interval == 0:
                engine.settle()
                engine.check_status()
                save_checkpoint(cfg.checkpoint_dir, model.to_host(), done, self.host_data.id, cfg.world_size)
                self.events.append("checkpoint", iteration=done)
            if cfg.metrics_dir and done % self.sampler.batches_per_epoch == 0:
                engine.settle()
                engine.check_status()
                self._record_epoch(done, model)
        engine.settle()
        engine.check_status()
        t1.record()
        torch.cuda.synchronize()
        span = t0.elapsed_time(t1) / 1e3
        losses = engine.loss_values()[start:]
        for i, l in enumerate(losses):
            if not np.isfinite(l):
                raise nnkit.NumericError(f"loss is not finite at iteration {start + i}: {l}")
        ledger = reader.ledger() if reader is not None else {"ok": True}
        if reader is not None:
            reader.close()
        hold = self.cfg.data.build_holdout()
        top1 = nnkit.evaluate(model, hold.samples, hold.labels, 1)
        top5 = nnkit.evaluate(model, hold.samples, hold.labels, min(5, self.classes))
        throughput = trained * cfg.train.batch_size / span if span > 0 else 0.0
        self.events.append("done", iterations=self.total_steps, top1=top1, top5=top5,
                           throughput=round(throughput, 3), ledger=ledger)
        self._flush_metrics()
        self.events.close()
        return StudentResult(cfg.rank, self.total_steps, 0, top1, top5, model.to_host(), ledger, throughput,
                             losses)

    def _initial_acquire(self, reader: DistilReader) -> None:
        want = self.cfg.teacher_count
        if want == "auto":
            got = reader.acquire(1)
            n = self._auto_teacher_count(reader) if got else 1
            if n > 1:
                reader.acquire(n - 1)
            self.events.append("static_schedule", teachers=n)
        else:
            reader.acquire(int(want))

    def _auto_teacher_count(self, reader: DistilReader) -> int:
        """Measure our step rate and one teacher's batch rate on the device,
        then size the set as ceil(t_s / t_t) (edl/student_node.py:807-833)."""
        dims = self._dims()
        model = Model.from_host(formats.init_model(dims, self.cfg.train.seed), self.dataset.device)
        cfg = self._train_config()
        B = self.cfg.train.batch_size
        eng = StudentStep(model, cfg, B)
        batch = self.sampler.batch_for(0, out=eng.batch)
        uniform = SoftLabels(torch.full((B, self.k), 1.0 / self.classes, device=model.device),
                             torch.arange(self.k, dtype=torch.int32, device=model.device).repeat(B, 1),
                             cfg.temperature)
        probes = 3
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        eng.step(batch, uniform if cfg.beta > 0 else None)
        s.record()
        for _ in range(probes):
            eng.step(batch, uniform if cfg.beta > 0 else None)
        e.record()
        e.synchronize()
        t_s = probes / max(s.elapsed_time(e) / 1e3, 1e-9)
        h = next(iter(reader._teachers.values()))
        tm = h.worker.model
        x = batch.inputs
        nnkit.teacher_soft_labels(tm, x, cfg.temperature, self.k)
        s.record()
        for _ in range(probes):
            nnkit.teacher_soft_labels(tm, x, cfg.temperature, self.k)
        e.record()
        e.synchronize()
        t_t = probes / max(s.elapsed_time(e) / 1e3, 1e-9)
        return static_schedule(ThroughputProfile(t_s=t_s, t_t=min(t_t, t_s * 64)))

    def _record_epoch(self, iteration: int, model: Model) -> None:
        hold = self.cfg.data.build_holdout()
        k5 = min(5, self.classes)
        self._epoch_rows.append({
            "iteration": iteration, "epoch": iteration // self.sampler.batches_per_epoch,
            "top1": round(nnkit.evaluate(model, hold.samples, hold.labels, 1), 4),
            "top5": round(nnkit.evaluate(model, hold.samples, hold.labels, k5), 4)})

    def _flush_metrics(self) -> None:
        if not self.cfg.metrics_dir or not self._epoch_rows:
            return
        path = os.path.join(self.cfg.metrics_dir, f"student-{self.cfg.rank}-epochs.csv")
        with open(path, "w", newline="") as fh:
            w = csv.DictWriter(fh, fieldnames=list(self._epoch_rows[0]))
            w.writeheader()
            w.writerows(self._epoch_rows)
