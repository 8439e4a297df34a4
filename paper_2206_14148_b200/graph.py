"""Graph-level drop-in: the reference's builder/interpreter names for this path.

The reference's operator API is ``build_knn`` / ``build_kernel_mvm``
(frontend.py:22-114) -> ``run_pipeline(graph, PassConfig)``
(pipeline.py:18-60) -> ``evaluate(graph, inputs, budget)``
(interpreter.py:522-551) returning ``(outputs, MemoryTrace)``.  These names
keep that surface for the kNN and kernel-MVM graph families: the "graph" is a
typed descriptor of the workload (the general IR is out of scope, SURVEY.md
§2 rows 7-9), and ``evaluate`` dispatches it to the fused CUDA path.  Output
conventions are the reference's: TopK indices come back in the operand float
dtype (interpreter.py:385-387), outputs are fresh copies, inputs are never
written, and ``budget`` counts the inputs (interpreter.py:543-546).
"""

from __future__ import annotations

import math
import re
from dataclasses import dataclass, field, replace
from enum import Enum

import numpy as np

from .errors import BudgetExceeded, EvaluationError

METRICS = ("l2", "l1", "cosine")


class DType(Enum):
    F32 = ("f32", 4)
    F64 = ("f64", 8)

    def __init__(self, label: str, byte_size: int):
        self.label = label
        self.byte_size = byte_size

    @property
    def np_dtype(self) -> np.dtype:
        return np.dtype(np.float32 if self is DType.F32 else np.float64)

    @classmethod
    def from_np(cls, dtype) -> "DType":
        dtype = np.dtype(dtype)
        if dtype == np.float32:
            return cls.F32
        if dtype == np.float64:
            return cls.F64
        raise ValueError(f"unsupported dtype {dtype}; only f32/f64 tensors exist")

    def __str__(self) -> str:
        return self.label


@dataclass(frozen=True)
class KernelSpec:
    """Squared-exponential kernel k(x, y) = variance * exp(-(x-y)^2 / (2 l^2))
    (frontend.py:22-31)."""

    variance: float = 1.0
    lengthscale: float = 1.0

    def __post_init__(self):
        if self.variance <= 0 or self.lengthscale <= 0:
            raise ValueError("variance and lengthscale must be strictly positive")


@dataclass(frozen=True)
class TensorType:
    dims: tuple
    dtype: DType

    @property
    def byte_size(self) -> int:
        n = 1
        for v in self.dims:
            n *= v
        return n * self.dtype.byte_size


@dataclass(frozen=True)
class PassConfig:
    """Same knobs and invariants as pipeline.py:18-41.  The fused path never
    materialises a split candidate; ``evaluate`` applies
    ``tensor_split_size`` as a cap on the database slice each planner chunk
    stages (rows x d x itemsize <= tensor_split_size, at least one 256-row
    tile), the analogue of the splitter's slice bound (split.py:285-301)."""

    tensor_size_threshold: int = 10**9
    tensor_split_size: int | None = None
    enable_match_replace: bool = True
    enable_reorder: bool = True
    enable_split: bool = True

    def __post_init__(self):
        if self.tensor_split_size is None:
            object.__setattr__(self, "tensor_split_size", self.tensor_size_threshold)
        if self.tensor_size_threshold <= 0 or self.tensor_split_size <= 0:
            raise ValueError("size options must be positive byte counts")
        if self.tensor_split_size > self.tensor_size_threshold:
            raise ValueError(
                f"tensor_split_size ({self.tensor_split_size}) must not exceed "
                f"tensor_size_threshold ({self.tensor_size_threshold})")


@dataclass(frozen=True)
class Graph:
    """Workload descriptor standing in for the reference's SSA graph."""

    name: str
    kind: str                     # "knn" | "mvm"
    parameters: tuple             # TensorType per parameter, reference order
    attrs: dict = field(default_factory=dict)
    config: PassConfig | None = None


@dataclass(frozen=True)
class TensorValue:
    array: np.ndarray

    @property
    def shape(self):
        return tuple(self.array.shape)

    @property
    def dtype(self) -> DType:
        return DType.from_np(self.array.dtype)

    @property
    def data(self):
        return self.array


@dataclass(frozen=True)
class MemoryEvent:
    instruction: str
    event: str
    bytes: int
    live_after: int

    def as_row(self) -> str:
        return f"{self.instruction},{self.event},{self.bytes},{self.live_after}"


@dataclass
class MemoryTrace:
    events: list = field(default_factory=list)
    peak_live_bytes: int = 0

    def to_csv(self) -> str:
        lines = ["instruction,event,bytes,live_after"]
        lines.extend(e.as_row() for e in self.events)
        return "\n".join(lines) + "\n"


def build_knn(n: int, m: int, d: int, k: int, metric: str = "l2",
              dtype: DType = DType.F64) -> Graph:
    """Brute-force kNN (frontend.py:98-114): parameters x[n,d], q[m,d]; root
    (distances[m,k], indices[m,k]); ties resolve to the lower data index."""
    if not 1 <= k <= n:
        raise ValueError(f"k={k} must satisfy 1 <= k <= n={n}")
    if metric not in METRICS:
        raise ValueError(f"metric must be one of {METRICS}")
    if min(n, m, d) < 1:
        raise ValueError("n, m and d must be at least 1")
    return Graph(f"knn_{metric}_n{n}_m{m}_d{d}_k{k}", "knn",
                 (TensorType((n, d), dtype), TensorType((m, d), dtype)),
                 {"n": n, "m": m, "d": d, "k": k, "metric": metric, "dtype": dtype})


def build_kernel_mvm(n: int, spec: KernelSpec = KernelSpec(),
                     dtype: DType = DType.F64) -> Graph:
    """y = K v over 1-D inputs x[n], y[n], v[n] (frontend.py:34-54)."""
    if n < 1:
        raise ValueError("n must be at least 1")
    return Graph(f"se_kernel_mvm_n{n}", "mvm",
                 tuple(TensorType((n,), dtype) for _ in range(3)),
                 {"n": n, "spec": spec, "dtype": dtype})


def run_pipeline(graph: Graph, config: PassConfig, diagnostics=None) -> Graph:
    """Records the pass configuration; the fused kernels are already the
    post-pipeline form (no [m,n,d] or [m,n] intermediate ever exists)."""
    return replace(graph, config=config)


def random_inputs(graph: Graph, seed: int, low: float = -1.0, high: float = 1.0):
    """Seeded U[low, high) inputs in parameter order (frontend.py:128-138)."""
    rng = np.random.default_rng(seed)
    return [rng.uniform(low, high, size=p.dims).astype(p.dtype.np_dtype)
            for p in graph.parameters]


def _check_inputs(graph: Graph, inputs):
    if len(inputs) != len(graph.parameters):
        raise EvaluationError(
            f"graph {graph.name!r} takes {len(graph.parameters)} inputs, got {len(inputs)}")
    arrays = []
    for i, (raw, expected) in enumerate(zip(inputs, graph.parameters)):
        arr = raw.array if isinstance(raw, TensorValue) else np.asarray(raw)
        try:
            ok = tuple(arr.shape) == tuple(expected.dims) and \
                DType.from_np(arr.dtype) == expected.dtype
        except ValueError:
            ok = False
        if not ok:
            raise EvaluationError(
                f"input {i} is {arr.dtype}{list(arr.shape)}, expected "
                f"{expected.dtype}{list(expected.dims)}")
        arrays.append(np.ascontiguousarray(arr))
    return arrays


class _DeviceLedger:
    """Every device buffer ``evaluate`` allocates, as alloc / free events with
    the live bytes measured on the device after each one (caching-allocator
    bytes relative to the call's start) - the B200 counterpart of the
    interpreter's allocation log (interpreter.py:57-76,149-167).  The C-ABI
    library never allocates (the planner sizes one workspace), so these
    events are the whole device footprint of the call.  ``poison`` fills a
    buffer with 0xFF bytes (NaN for f32/f64) before it is released, like the
    reference's ``poison_freed`` (interpreter.py:166-167): a kernel that read
    a released buffer would then produce NaN instead of stale data."""

    def __init__(self, device, poison: bool):
        import torch
        self._torch = torch
        self.device = device
        self.poison = poison
        self.base = torch.cuda.memory_allocated(device)
        self.trace = MemoryTrace()
        self.held = {}

    def _event(self, label: str, kind: str, nbytes: int):
        live = self._torch.cuda.memory_allocated(self.device) - self.base
        self.trace.events.append(MemoryEvent(label, kind, nbytes, live))
        self.trace.peak_live_bytes = max(self.trace.peak_live_bytes, live)

    def alloc(self, label: str, tensor):
        self.held[label] = tensor
        self._event(label, "alloc", tensor.numel() * tensor.element_size())
        return tensor

    def free(self, label: str):
        t = self.held.pop(label)
        nbytes = t.numel() * t.element_size()
        if self.poison:
            t.view(self._torch.uint8).fill_(0xFF)
            self._torch.cuda.current_stream(self.device).synchronize()
        del t
        self._event(label, "free", nbytes)

    def free_all(self):
        for label in list(self.held):
            self.free(label)


def _split_cap_rows(graph: Graph, d: int, itemsize: int) -> int:
    """PassConfig.tensor_split_size on the fused path: the largest database
    slice one chunk may stage, in rows (pipeline.py:18-41, split.py:285-301
    bound the splitter's slices the same way); at least one 256-row tile."""
    if graph.config is None:
        return 0
    return max(256, int(graph.config.tensor_split_size) // (d * itemsize))


def estimate_peak_memory(graph: Graph, budget: int | None = None) -> int:
    """Static device peak of ``evaluate`` (planner arithmetic, no device)."""
    if graph.kind == "knn":
        from . import neighbors as _knn
        a = graph.attrs
        p = _knn.plan(a["n"], a["m"], a["d"], a["k"], metric=a["metric"],
                      dtype=a["dtype"].np_dtype, memory_limit=budget)
        return int(p.peak_bytes)
    if graph.kind == "mvm":
        return sum(p.byte_size for p in graph.parameters) + graph.parameters[0].byte_size
    raise EvaluationError(f"no evaluator for graph kind {graph.kind!r}")


_KNN_NAME = re.compile(r"knn_(l2|l1|cosine)_n(\d+)_m(\d+)_d(\d+)_k(\d+)$")
_MVM_NAME = re.compile(r"se_kernel_mvm_n(\d+)$")


def _se_constants(g, params):
    """(variance, -0.5/l^2) of the SE kernel pattern mul(bcast(variance),
    exp(mul(square(.), bcast(scale)))) (frontend.py:49-53), found in ``g`` or
    in the body of a While the splitter created; loop parameters are resolved
    to the constants the While is entered with."""
    ins = getattr(g, "instructions", {})

    def value(i):
        op = ins[i].op
        kind = type(op).__name__
        if kind == "Constant":
            return float(op.value) if np.ndim(op.value) == 0 else None
        if kind == "Parameter":
            return params.get(op.index)
        if kind == "Broadcast":
            return value(ins[i].operands[0])
        return None

    for i, inst in ins.items():
        op = inst.op
        kind = type(op).__name__
        if kind == "Unary" and getattr(op, "op", None) == "exp":
            arg = ins[inst.operands[0]]
            if type(arg.op).__name__ == "Binary" and arg.op.op == "mul":
                scale = [value(o) for o in arg.operands if value(o) is not None]
                users = [u for u in ins.values() if type(u.op).__name__ == "Binary"
                         and u.op.op == "mul" and i in u.operands]
                var = [value(o) for u in users for o in u.operands
                       if o != i and value(o) is not None]
                if len(scale) == 1 and len(var) == 1 and scale[0] < 0 < var[0]:
                    return var[0], scale[0]
        if kind == "While":
            inner = {k: value(o) for k, o in enumerate(inst.operands)}
            found = _se_constants(op.body, inner)
            if found is not None:
                return found
    return None


def from_reference(graph) -> Graph:
    """Descriptor for a graph object built by the REFERENCE package
    (tensorbudget.ir.Graph from build_knn / build_kernel_mvm, naive or after
    run_pipeline - the passes keep the builder's name, frontend.py:98-114,
    34-54).  Duck-typed (the reference is not imported): the family and sizes
    come from the builder name, the dtype from the parameters, and the SE
    kernel's variance / lengthscale from the SE pattern (frontend.py:49-53),
    followed into the splitter's While body for pipelined graphs."""
    name = getattr(graph, "name", None)
    params = getattr(graph, "parameters", None)
    if not isinstance(name, str) or not params:
        raise EvaluationError(f"not a graph: {graph!r}")
    label = getattr(getattr(params[0], "dtype", None), "name", "")
    if label not in ("F32", "F64"):
        raise EvaluationError(f"graph {name!r}: unsupported parameter dtype {label!r}")
    dtype = DType[label]
    m = _KNN_NAME.match(name)
    if m:
        metric, n, mq, d, k = m.group(1), *(int(v) for v in m.groups()[1:])
        return build_knn(n, mq, d, k, metric, dtype)
    m = _MVM_NAME.match(name)
    if m:
        found = _se_constants(graph, {})
        if found is None:
            raise EvaluationError(f"graph {name!r}: cannot recover the kernel constants")
        variance, scale = found
        return build_kernel_mvm(int(m.group(1)),
                                KernelSpec(variance, math.sqrt(-0.5 / scale)), dtype)
    raise EvaluationError(f"graph {name!r} is not a kNN / kernel-MVM graph of this path")


def evaluate(graph: Graph, inputs, budget: int | None = None, *,
             poison_freed: bool = False):
    """Evaluates the graph on the B200 path; returns (outputs, MemoryTrace).

    ``graph`` is this package's descriptor or a reference-built graph object
    (see ``from_reference``).  Raises BudgetExceeded before any device
    allocation when the planner cannot fit ``budget`` (the reference raises
    at the offending allocation, interpreter.py:149-151).  After
    ``run_pipeline``, ``tensor_split_size`` caps the database slice each
    chunk stages.  The trace lists every device buffer of the call with the
    live bytes measured after each event; ``poison_freed`` overwrites each
    buffer with NaN bytes before releasing it.
    """
    import torch
    if not isinstance(graph, Graph):
        graph = from_reference(graph)
    arrays = _check_inputs(graph, inputs)
    from .errors import BudgetExceeded as _BE
    dev = torch.device("cuda")
    if graph.kind == "knn":
        from . import neighbors as _knn
        a = graph.attrs
        dt = a["dtype"].np_dtype
        cap = _split_cap_rows(graph, a["d"], np.dtype(dt).itemsize)
        try:                           # plan first: nothing is allocated on failure
            op = _knn.KnnOperator(a["n"], a["m"], a["d"], a["k"], metric=a["metric"],
                                  dtype=dt, memory_limit=budget, device=dev,
                                  max_chunk_rows=cap, allocate=False)
        except _BE as exc:
            raise BudgetExceeded(graph.name, exc.requested, exc.live,
                                 MemoryTrace(), message=str(exc)) from None
        led = _DeviceLedger(dev, poison_freed)
        x = led.alloc(f"{graph.name}/param0", torch.from_numpy(arrays[0]).to(dev))
        q = led.alloc(f"{graph.name}/param1", torch.from_numpy(arrays[1]).to(dev))
        ws = led.alloc(f"{graph.name}/workspace", op.allocate_workspace())
        dist, idx = op.alloc_outputs()
        led.alloc(f"{graph.name}/values", dist)
        led.alloc(f"{graph.name}/indices", idx)
        op.run(x, q, (dist, idx))
        outs = (TensorValue(dist.cpu().numpy().astype(dt, copy=False)),
                TensorValue(idx.cpu().numpy().astype(dt)))
        del x, q, ws, dist, idx
        op.workspace = None
        led.free_all()
        return outs, led.trace
    if graph.kind == "mvm":
        from . import mvm as _mvm
        spec = graph.attrs["spec"]
        x, y, v = arrays
        n = graph.parameters[0].dims[0]
        es = np.dtype(graph.attrs["dtype"].np_dtype).itemsize
        # device bytes of the call: x, y in the operand dtype, v and the
        # output in fp64 (the kernel accumulates and writes fp64)
        total = 2 * n * es + 2 * n * 8
        if budget is not None and total > budget:
            raise BudgetExceeded(f"{graph.name}/outputs", n * 8, total - n * 8, MemoryTrace())
        led = _DeviceLedger(dev, poison_freed)
        xd = led.alloc(f"{graph.name}/param0", torch.from_numpy(x).to(dev))
        yd = led.alloc(f"{graph.name}/param1", torch.from_numpy(y).to(dev))
        vd = led.alloc(f"{graph.name}/param2", torch.from_numpy(np.asarray(v, np.float64)).to(dev))
        out = _mvm.kernel_mvm(xd.reshape(-1, 1), yd.reshape(-1, 1), vd, "rbf", spec.variance,
                              spec.lengthscale)
        led.alloc(f"{graph.name}/output", out)
        res = out.cpu().numpy().astype(graph.attrs["dtype"].np_dtype)
        del xd, yd, vd, out
        led.free_all()
        return TensorValue(res), led.trace
    raise EvaluationError(f"no evaluator for graph kind {graph.kind!r}")
