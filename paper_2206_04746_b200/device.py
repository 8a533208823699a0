"""Device-resident pipeline: HBM-resident data, torch for memory/streams/NCCL.

torch provides device allocations, the CUDA stream and torch.distributed
(NCCL over NVLink) — plumbing only. Every computation is a libhvb200 kernel
called through the C ABI `hv_dev_*` entry points on torch's current stream.

Multi-GPU (north star): datapoints are sharded across ranks.
Encode and predict need no collective (codebooks and class vectors are
replicated). Classical training all-reduces the C x 32W uint32 class counts
and the C class row counts (one NCCL all-reduce each, bit-exact because
integer addition is associative). Online training in data-parallel "delta"
mode all-reduces each batch's per-class fp64 updates.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import torch

from . import _native as N

I32 = torch.int32


def _ptr(t: torch.Tensor | None):
    return None if t is None else C.c_void_p(t.data_ptr())


def _rows_view(t: torch.Tensor, W: int) -> int:
    """Row pitch (in words) of a (rows, W) int32 matrix view whose words are
    contiguous within a row; rejects anything else."""
    if t.dim() != 2 or t.shape[1] != W or (t.shape[0] > 1 and t.stride(1) != 1) or t.stride(0) < W:
        raise ValueError(f"expected a (rows, {W}) int32 row view with unit word stride, got shape "
                         f"{tuple(t.shape)} strides {t.stride()}")
    return t.stride(0)


def _contig_rows(t: torch.Tensor, W: int, what: str) -> None:
    if _rows_view(t, W) != W and t.shape[0] > 1:
        raise ValueError(f"{what}: needs unpitched (contiguous) rows; got row stride {t.stride(0)}")


def words_per_row(dim: int) -> int:
    return (dim + 31) // 32


def bins_pitch(features: int) -> int:
    """Row pitch of device uint8 bins (64-byte multiple, required by the fast encoder)."""
    return (features + 63) // 64 * 64


class DeviceContext:
    """hv_context bound to torch's current CUDA stream on `device`."""

    def __init__(self, device: int = 0):
        self.device = device
        self.ctx = N.context(device)
        self.bind()

    def bind(self, stream: torch.cuda.Stream | None = None):
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        # torch's default stream is the legacy NULL stream; hand the library
        # cudaStreamLegacy (0x1) explicitly so its kernels order with torch's.
        self.ctx.set_stream(s.cuda_stream or 0x1)
        return self

    @property
    def h(self):
        return self.ctx.handle

    def check(self):
        self.ctx.dev_check()


@dataclass
class DeviceCodebook:
    features: int
    bins: int
    dim: int
    id_vectors: torch.Tensor      # F x W int32 (uint32 bit patterns)
    value_vectors: torch.Tensor   # B x W
    encode_tiebreak: torch.Tensor  # W
    model_tiebreak: torch.Tensor   # W
    binding: int = N.BIND_ID_LEVEL

    @classmethod
    def make(cls, features: int, bins: int, dim: int, seed: int, device: int = 0,
             generation: int = N.GEN_RANDOM, binding: int = N.BIND_ID_LEVEL):
        """Seed substreams as the reference's build_context (experiment.cpp:119-144):
        codebook derive(seed,1), encode tiebreak derive(seed,2), model tiebreak derive(seed,3)."""
        import numpy as np

        L = N.lib()
        w = words_per_row(dim)
        idv = np.zeros((features, w), np.uint32)
        val = np.zeros((bins, w), np.uint32)
        N.check(L.hv_make_codebook(generation, features, bins, dim, L.hv_derive_seed(seed, 1),
                                   idv.ctypes.data_as(C.c_void_p), val.ctypes.data_as(C.c_void_p)))
        etb = np.zeros(w, np.uint32)
        mtb = np.zeros(w, np.uint32)
        N.check(L.hv_generate_random(1, dim, L.hv_derive_seed(seed, 2), etb.ctypes.data_as(C.c_void_p)))
        N.check(L.hv_generate_random(1, dim, L.hv_derive_seed(seed, 3), mtb.ctypes.data_as(C.c_void_p)))
        dev = torch.device("cuda", device)
        t = lambda a: torch.from_numpy(a.view(np.int32)).to(dev)
        return cls(features, bins, dim, t(idv), t(val), t(etb), t(mtb), binding)


class Engine:
    """Device-resident encode / classical train / online train / predict for one GPU."""

    def __init__(self, codebook: DeviceCodebook, classes: int, device: int = 0):
        self.cb = codebook
        self.C = classes
        self.D = codebook.dim
        self.W = words_per_row(codebook.dim)
        self.dc = DeviceContext(device)
        self.dev = torch.device("cuda", device)

    # -- data ----------------------------------------------------------------
    def synth(self, row0: int, rows: int, label_kind: int, data_seed: int):
        ldb = bins_pitch(self.cb.features)
        bins8 = torch.empty((rows, ldb), dtype=torch.uint8, device=self.dev)
        labels = torch.empty(rows, dtype=I32, device=self.dev)
        N.check(N.lib().hv_dev_synth(self.dc.h, row0, rows, self.cb.features, self.C, self.cb.bins, label_kind,
                                     data_seed, _ptr(bins8), ldb, _ptr(labels)))
        return bins8, labels

    def narrow(self, bins32: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
        rows = bins32.shape[0]
        ldb = bins_pitch(self.cb.features)
        if out is None:
            out = torch.empty((rows, ldb), dtype=torch.uint8, device=self.dev)
        N.check(N.lib().hv_dev_narrow_bins(self.dc.h, _ptr(bins32), rows, self.cb.features, self.cb.bins,
                                           _ptr(out), ldb))
        return out

    # -- encode --------------------------------------------------------------
    def pitched_empty(self, rows: int) -> torch.Tensor:
        """(rows, W) int32 view of rows padded to hv_row_pitch_words(D) words
        (16-byte rows: uint4 / TMA row reads in class counts and predict)."""
        ldw = N.lib().hv_row_pitch_words(self.D)
        return torch.empty((rows, ldw), dtype=I32, device=self.dev)[:, :self.W]

    def encode(self, bins8: torch.Tensor, out: torch.Tensor | None = None, pitched: bool = False) -> torch.Tensor:
        """Encode uint8 bins; `out` (or a new tensor, pitched if asked) may have
        any row stride >= W — the encoder writes words [0, W) of each row."""
        rows, ldb = bins8.shape
        if out is None:
            out = self.pitched_empty(rows) if pitched else torch.empty((rows, self.W), dtype=I32, device=self.dev)
        if out.stride(0) == self.W:
            N.check(N.lib().hv_dev_encode(self.dc.h, _ptr(bins8), ldb, rows, self.cb.features,
                                          _ptr(self.cb.id_vectors), _ptr(self.cb.value_vectors), self.cb.bins, self.D,
                                          self.cb.binding, _ptr(self.cb.encode_tiebreak), _ptr(out)))
        else:
            _rows_view(out, self.W)
            N.check(N.lib().hv_dev_encode_words(self.dc.h, _ptr(bins8), ldb, rows, self.cb.features,
                                                _ptr(self.cb.id_vectors), _ptr(self.cb.value_vectors), self.cb.bins,
                                                self.D, self.cb.binding, _ptr(self.cb.encode_tiebreak), 0, self.W,
                                                _ptr(out), out.stride(0)))
        return out

    def encode_words(self, bins8: torch.Tensor, word_begin: int, words: int,
                     out: torch.Tensor | None = None) -> torch.Tensor:
        """Encode only output words [word_begin, word_begin + words) of every row
        (the column slice a rank owns in D-sliced training)."""
        rows, ldb = bins8.shape
        if out is None:
            out = torch.empty((rows, words), dtype=I32, device=self.dev)
        N.check(N.lib().hv_dev_encode_words(self.dc.h, _ptr(bins8), ldb, rows, self.cb.features,
                                            _ptr(self.cb.id_vectors), _ptr(self.cb.value_vectors), self.cb.bins,
                                            self.D, self.cb.binding, _ptr(self.cb.encode_tiebreak), word_begin,
                                            words, _ptr(out), out.stride(0)))
        return out

    # -- classical -----------------------------------------------------------
    def zero_counts(self):
        return (torch.zeros((self.C, 32 * self.W), dtype=I32, device=self.dev),
                torch.zeros(self.C, dtype=torch.int64, device=self.dev))

    def class_counts(self, enc: torch.Tensor, labels: torch.Tensor, counts: torch.Tensor, class_rows: torch.Tensor):
        ldw = _rows_view(enc, self.W)
        N.check(N.lib().hv_dev_class_counts_pitched(self.dc.h, _ptr(enc), ldw, enc.shape[0], self.D, _ptr(labels),
                                                    self.C, _ptr(counts), _ptr(class_rows)))

    def binarize(self, counts: torch.Tensor, class_rows: torch.Tensor, out: torch.Tensor | None = None):
        if out is None:
            out = torch.empty((self.C, self.W), dtype=I32, device=self.dev)
        N.check(N.lib().hv_dev_binarize_counts(self.dc.h, _ptr(counts), _ptr(class_rows), self.C, self.D,
                                               _ptr(self.cb.model_tiebreak), _ptr(out)))
        return out

    def train_classical(self, enc: torch.Tensor, labels: torch.Tensor, group=None):
        """Per-shard counts, then (if distributed) one all-reduce each, then binarise."""
        counts, rows = self.zero_counts()
        self.class_counts(enc, labels, counts, rows)
        if group is not None or (torch.distributed.is_available() and torch.distributed.is_initialized()
                                 and torch.distributed.get_world_size() > 1):
            torch.distributed.all_reduce(counts, group=group)
            torch.distributed.all_reduce(rows, group=group)
        cv = self.binarize(counts, rows)
        return cv, counts, rows

    # -- predict -------------------------------------------------------------
    def predict(self, cv: torch.Tensor, enc: torch.Tensor, labels: torch.Tensor | None = None,
                distances: torch.Tensor | None = None, popcounts: torch.Tensor | None = None):
        rows = enc.shape[0]
        if labels is None:
            labels = torch.empty(rows, dtype=I32, device=self.dev)
        ldw = _rows_view(enc, self.W)
        N.check(N.lib().hv_dev_predict_hamming_pitched(self.dc.h, _ptr(cv), self.C, self.D, _ptr(enc), ldw, rows,
                                                       _ptr(labels), _ptr(distances), _ptr(popcounts)))
        return labels

    # -- online --------------------------------------------------------------
    def train_online(self, enc: torch.Tensor, labels: torch.Tensor, batch_size: int, gamma: float = 1.0):
        """Exact single-GPU online training (bit-identical to the reference)."""
        _contig_rows(enc, self.W, "train_online")
        acc = torch.empty((self.C, self.D), dtype=torch.float64, device=self.dev)
        weight = torch.empty(self.C, dtype=torch.float64, device=self.dev)
        counts = torch.empty(self.C, dtype=torch.int64, device=self.dev)
        cv = torch.empty((self.C, self.W), dtype=I32, device=self.dev)
        N.check(N.lib().hv_dev_train_online(self.dc.h, _ptr(enc), enc.shape[0], self.D, _ptr(labels), self.C,
                                            batch_size, gamma, _ptr(self.cb.model_tiebreak), _ptr(acc), _ptr(weight),
                                            _ptr(counts), _ptr(cv)))
        return acc, weight, counts, cv

    def train_online_sharded(self, enc_shard: torch.Tensor, labels_shard: torch.Tensor, global_rows: int,
                             batch_size: int, rank: int, world: int, gamma: float = 1.0, group=None):
        """Data-parallel online training (delta mode).

        Global batch b covers global rows [b*B, (b+1)*B); rank r owns the r-th
        contiguous slice of every batch (`shard_rows_online`). Each rank scores
        its slice against the replicated class vectors, forms per-class fp64
        deltas in sample order, the deltas are all-reduced and applied
        identically everywhere. The bootstrap classical pass on batch 0 is an
        all-reduced count like train_classical.
        """
        _contig_rows(enc_shard, self.W, "train_online_sharded")
        import torch.distributed as dist

        # bootstrap: classical on global batch 0
        first = min(batch_size, global_rows)
        lo, hi = online_slice(0, first, rank, world)
        counts, rows = self.zero_counts()
        self.class_counts(enc_shard[:hi - lo], labels_shard[:hi - lo], counts, rows)
        if world > 1:
            dist.all_reduce(counts, group=group)
            dist.all_reduce(rows, group=group)
        acc = counts[:, : self.D].to(torch.float64).contiguous()
        weight = rows.to(torch.float64)
        cnt = rows.clone()
        cv = self.binarize(counts, rows)
        d_acc = torch.empty_like(acc)
        d_w = torch.empty_like(weight)
        d_c = torch.empty_like(cnt)
        touched = torch.empty(self.C, dtype=I32, device=self.dev)
        off = 0
        for start in range(0, global_rows, batch_size):
            n = min(batch_size, global_rows - start)
            lo, hi = online_slice(start, n, rank, world)
            k = hi - lo
            N.check(N.lib().hv_dev_online_delta(self.dc.h, _ptr(cv), self.C, self.D, _ptr(enc_shard[off:off + k]), k,
                                                _ptr(labels_shard[off:off + k]), gamma, _ptr(d_acc), _ptr(d_w),
                                                _ptr(d_c), _ptr(touched)))
            off += k
            if world > 1:
                dist.all_reduce(d_acc, group=group)
                dist.all_reduce(d_w, group=group)
                dist.all_reduce(d_c, group=group)
                dist.all_reduce(touched, group=group)
            N.check(N.lib().hv_dev_apply_online_delta(self.dc.h, self.C, self.D, _ptr(d_acc), _ptr(d_w), _ptr(d_c),
                                                      _ptr(touched), _ptr(self.cb.model_tiebreak), _ptr(acc),
                                                      _ptr(weight), _ptr(cnt), _ptr(cv)))
        return acc, weight, cnt, cv


class PeerShared:
    """One device buffer per rank shared with every peer through CUDA IPC:
    two payload slots (epoch parity) and `world` uint32 arrival flags. Ranks
    add their contributions straight into every rank's slot of the current
    parity (system-scope atomics over NVLink P2P), release-store the epoch into
    every peer's flag, and acquire-wait for all flags (csrc/hv_peer.cu).

    `local_ranks` (tests): base pointers of zeroed buffers of `nbytes` for
    ranks emulated in one process; normally buffers come from hv_shared_alloc
    plus an all_gather of the IPC handles.
    """

    def __init__(self, engine: "Engine", rank: int, world: int, payload_bytes: int, group=None, local_ranks=None):
        import ctypes as _C
        import torch.distributed as dist

        self.e, self.rank, self.world = engine, rank, world
        self.slot = self.slot_bytes(payload_bytes)
        self.off_flags = 2 * self.slot
        L = N.lib()
        self._owned, self._opened = [], []
        if local_ranks is not None:
            bases = list(local_ranks)
        else:
            hs = L.hv_shared_handle_size()
            base = _C.c_void_p()
            handle = (_C.c_uint8 * hs)()
            N.check(L.hv_shared_alloc(engine.dc.h, self.nbytes(payload_bytes, world), _C.byref(base), handle))
            self._owned.append(base.value)
            handles = [None] * world
            dist.all_gather_object(handles, bytes(handle), group=group)
            bases = []
            for q in range(world):
                if q == rank:
                    bases.append(base.value)
                    continue
                ptr = _C.c_void_p()
                N.check(L.hv_shared_open(engine.dc.h, (_C.c_uint8 * hs).from_buffer_copy(handles[q]), _C.byref(ptr)))
                self._opened.append(ptr.value)
                bases.append(ptr.value)
        self.bases = bases
        dev = engine.dev
        self.flags_ptrs = torch.tensor([b_ + self.off_flags for b_ in bases], dtype=torch.int64, device=dev)
        self._ptrs = {}
        if local_ranks is None and world > 1:
            torch.cuda.synchronize(dev)
            dist.barrier(group=group)  # every buffer is zeroed and open before anyone adds into it

    @staticmethod
    def slot_bytes(payload_bytes: int) -> int:
        return (payload_bytes + 255) // 256 * 256

    @classmethod
    def nbytes(cls, payload_bytes: int, world: int) -> int:
        return 2 * cls.slot_bytes(payload_bytes) + 4 * world

    def peer_ptrs(self, par: int, offset: int = 0) -> torch.Tensor:
        """Device array of every rank's address of (parity slot + offset)."""
        key = (par, offset)
        if key not in self._ptrs:
            self._ptrs[key] = torch.tensor([b_ + par * self.slot + offset for b_ in self.bases], dtype=torch.int64,
                                           device=self.e.dev)
        return self._ptrs[key]

    def own(self, par: int, offset: int, shape, dtype) -> torch.Tensor:
        return _wrap(self.bases[self.rank] + par * self.slot + offset, shape, dtype, self.e.dev)

    def signal(self, epoch: int):
        N.check(N.lib().hv_dev_signal_peers(self.e.dc.h, _ptr(self.flags_ptrs), self.world, self.rank, epoch))

    def wait(self, epoch: int):
        N.check(N.lib().hv_dev_wait_peers(self.e.dc.h, C.c_void_p(self.bases[self.rank] + self.off_flags),
                                          self.world, epoch))

    def zero(self, par: int, nbytes: int):
        self.own(par, 0, (nbytes,), torch.uint8).zero_()

    def close(self):
        L = N.lib()
        for p_ in self._opened:
            L.hv_shared_close(self.e.dc.h, C.c_void_p(p_))
        for p_ in self._owned:
            L.hv_shared_free(self.e.dc.h, C.c_void_p(p_))
        self._opened, self._owned = [], []


class PeerCounts(PeerShared):
    """Classical class counts fused with their all-reduce over peer memory:
    `count` adds this rank's exact per-bit class counts and class row counts
    into every rank's buffer and signals; `wait` returns the global counts;
    `release` zeroes the parity slot once the caller has binarised it."""

    def __init__(self, engine: "Engine", rank: int, world: int, group=None, local_ranks=None):
        self.nc = engine.C * 32 * engine.W
        self.off_rows = (self.nc * 4 + 7) // 8 * 8
        super().__init__(engine, rank, world, self.payload(engine), group, local_ranks)
        self.epoch = 0

    @staticmethod
    def payload(engine: "Engine") -> int:
        nc = engine.C * 32 * engine.W
        return (nc * 4 + 7) // 8 * 8 + 8 * engine.C

    @classmethod
    def buffer_bytes(cls, engine: "Engine", world: int) -> int:
        return cls.nbytes(cls.payload(engine), world)

    def own_counts(self, par: int):
        e = self.e
        return (self.own(par, 0, (e.C, 32 * e.W), torch.int32), self.own(par, self.off_rows, (e.C,), torch.int64))

    def count(self, enc: torch.Tensor, labels: torch.Tensor) -> int:
        self.epoch += 1
        par = self.epoch & 1
        ldw = _rows_view(enc, self.e.W)
        N.check(N.lib().hv_dev_class_counts_peers_pitched(self.e.dc.h, _ptr(enc), ldw, enc.shape[0], self.e.D,
                                                          _ptr(labels), self.e.C, _ptr(self.peer_ptrs(par)),
                                                          _ptr(self.peer_ptrs(par, self.off_rows)), self.world))
        self.signal(self.epoch)
        return self.epoch

    def wait(self, epoch: int):  # noqa: D102 - returns this rank's global counts of the epoch
        PeerShared.wait(self, epoch)
        return self.own_counts(epoch & 1)

    def reduce(self, enc: torch.Tensor, labels: torch.Tensor):
        return self.wait(self.count(enc, labels))

    def release(self, epoch: int):
        self.zero(epoch & 1, self.payload(self.e))


class PeerPopc(PeerShared):
    """The per-batch popcount all-reduce of word-sliced online training fused
    into the partial-popcount kernel (hv_dev_online_partial_popc_peers)."""

    def __init__(self, engine: "Engine", rank: int, world: int, batch_size: int, group=None, local_ranks=None):
        self.bsz = batch_size
        self.epoch = 0
        super().__init__(engine, rank, world, self.payload(engine, batch_size), group, local_ranks)

    def next_epoch(self) -> int:
        """Epochs must grow across runs: a peer's flag passes wait(e) once it
        holds any epoch >= e, so restarting at 1 would skip the wait."""
        self.epoch += 1
        return self.epoch

    @staticmethod
    def payload(engine: "Engine", batch_size: int) -> int:
        return 4 * batch_size * engine.C

    @classmethod
    def buffer_bytes(cls, engine: "Engine", batch_size: int, world: int) -> int:
        return cls.nbytes(cls.payload(engine, batch_size), world)

    def partial(self, cv: torch.Tensor, words: int, batch: torch.Tensor, n: int, epoch: int):
        par = epoch & 1
        N.check(N.lib().hv_dev_online_partial_popc_peers(self.e.dc.h, _ptr(cv), self.e.C, words, _ptr(batch), n,
                                                         _ptr(self.peer_ptrs(par)), self.world))
        self.signal(epoch)

    def summed(self, epoch: int, n: int) -> torch.Tensor:
        PeerShared.wait(self, epoch)
        return self.own(epoch & 1, 0, (n, self.e.C), torch.int32)

    def release(self, epoch: int):
        self.zero(epoch & 1, self.payload(self.e, self.bsz))


def _wrap(ptr: int, shape, dtype, device):
    """A torch view of raw device memory (no ownership)."""
    class _CAI:
        def __init__(self):
            typestr = {torch.int32: "<i4", torch.int64: "<i8", torch.float64: "<f8", torch.uint8: "|u1"}[dtype]
            self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr, "data": (ptr, False),
                                             "version": 3, "strides": None, "stream": None}

    return torch.as_tensor(_CAI(), device=device)


class DSlicedOnline:
    """Exact multi-GPU online training by output-word slices.

    Rank r owns words [w0, w0 + words) of every hypervector (`word_slice`) and
    the matching columns of the fp64 accumulators; class weights and counts
    are replicated. Per batch the only collective is the all-reduce of the
    rows x C partial Hamming popcounts, after which every rank derives the
    same predictions and deltas and replays the reference's sample-ordered
    in-place additions (model.cpp:54-63, 250-280) on its own columns — so
    accumulators, class vectors and labels are bit-identical to the
    single-GPU trainer for any number of ranks.

    `enc_slice` is this rank's rows x words slice of ALL rows (Engine.encode_words);
    labels are replicated.
    """

    def __init__(self, engine: "Engine", enc_slice: torch.Tensor, labels: torch.Tensor, batch_size: int, w0: int,
                 gamma: float = 1.0):
        if batch_size < 1:
            raise ValueError("train_online: batch_size must be >= 1")
        self.e, self.enc, self.labels = engine, enc_slice, labels
        self.rows, self.words = enc_slice.shape
        self.bsz, self.w0, self.gamma = batch_size, w0, gamma
        e = engine
        self.slice_bits = min(e.D, 32 * (w0 + self.words)) - 32 * w0
        self.acc = torch.empty((e.C, self.slice_bits), dtype=torch.float64, device=e.dev)
        self.weight = torch.empty(e.C, dtype=torch.float64, device=e.dev)
        self.counts = torch.empty(e.C, dtype=torch.int64, device=e.dev)
        self.cv = torch.empty((e.C, self.words), dtype=I32, device=e.dev)
        self.popc = torch.empty((min(batch_size, max(self.rows, 1)), e.C), dtype=I32, device=e.dev)
        first = min(batch_size, self.rows)
        N.check(N.lib().hv_dev_online_slice_init(e.dc.h, _ptr(enc_slice), first, _ptr(labels), e.C, e.D, w0,
                                                 self.words, _ptr(e.cb.model_tiebreak), _ptr(self.acc),
                                                 _ptr(self.weight), _ptr(self.counts), _ptr(self.cv)))

    def batches(self):
        return [(s, min(self.bsz, self.rows - s)) for s in range(0, self.rows, self.bsz)]

    def partial(self, start: int, n: int) -> torch.Tensor:
        """This rank's partial popcounts of batch [start, start+n) (to be summed over ranks)."""
        e = self.e
        out = self.popc[:n]
        N.check(N.lib().hv_dev_online_partial_popc(e.dc.h, _ptr(self.cv), e.C, self.words,
                                                   _ptr(self.enc[start:start + n]), n, _ptr(out)))
        return out

    def update(self, start: int, n: int, popc: torch.Tensor):
        e = self.e
        N.check(N.lib().hv_dev_online_slice_update(e.dc.h, _ptr(popc), e.C, e.D, self.w0, self.words,
                                                   _ptr(self.enc[start:start + n]), n,
                                                   _ptr(self.labels[start:start + n]), self.gamma,
                                                   _ptr(e.cb.model_tiebreak), _ptr(self.acc), _ptr(self.weight),
                                                   _ptr(self.counts), _ptr(self.cv)))

    def run(self, group=None, peers: "PeerPopc | None" = None):
        """All batches. With `peers` the popcount all-reduce is fused into the
        partial kernel over peer memory; otherwise, with >1 torch.distributed
        rank, the popcounts are all-reduced (NCCL)."""
        if peers is not None:
            # every batch enqueued by one library call (no per-batch host round trip)
            e, nb = self.e, len(self.batches())
            own = peers.bases[peers.rank]
            N.check(N.lib().hv_dev_online_sliced_run_peers(
                e.dc.h, _ptr(self.enc), self.rows, self.words, self.w0, e.D, _ptr(self.labels), e.C, self.bsz,
                self.gamma, _ptr(e.cb.model_tiebreak), _ptr(peers.peer_ptrs(0)), _ptr(peers.peer_ptrs(1)),
                C.c_void_p(own), C.c_void_p(own + peers.slot), _ptr(peers.flags_ptrs),
                C.c_void_p(own + peers.off_flags), peers.world, peers.rank, peers.epoch, _ptr(self.acc),
                _ptr(self.weight), _ptr(self.counts), _ptr(self.cv)))
            peers.epoch += nb
            return self.acc, self.weight, self.counts, self.cv
        dist = torch.distributed
        multi = dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1
        for start, n in self.batches():
            p = self.partial(start, n)
            if multi:
                dist.all_reduce(p, group=group)
            self.update(start, n, p)
        return self.acc, self.weight, self.counts, self.cv

    def peer_partial(self, peers: "PeerPopc", start: int, n: int, epoch: int):
        """Add this rank's partial popcounts of a batch into every rank's buffer and signal."""
        peers.partial(self.cv, self.words, self.enc[start:start + n], n, epoch)

    def peer_update(self, peers: "PeerPopc", start: int, n: int, epoch: int):
        """Wait for every rank's partials, apply the batch, free the parity slot."""
        self.update(start, n, peers.summed(epoch, n))
        peers.release(epoch)


# ------------------------------------------------------------ sharding --
def word_slice(words: int, rank: int, world: int) -> tuple[int, int]:
    """Balanced contiguous split of a row's words: (first word, word count) of `rank`."""
    base, extra = divmod(words, world)
    w0 = rank * base + min(rank, extra)
    return w0, base + (1 if rank < extra else 0)


def shard_range(rows: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous row shard of rank `rank` (the GPU analogue of parallel_rows, parallel.cpp:10-36)."""
    chunk = (rows + world - 1) // world
    lo = min(rows, rank * chunk)
    return lo, min(rows, lo + chunk)


def online_slice(start: int, n: int, rank: int, world: int) -> tuple[int, int]:
    """Global rows of batch [start, start+n) owned by `rank` (contiguous split of the batch)."""
    lo, hi = shard_range(n, rank, world)
    return start + lo, start + hi


def shard_rows_online(global_rows: int, batch_size: int, rank: int, world: int) -> list[int]:
    """All global row indices a rank owns in data-parallel online training, in order."""
    out: list[int] = []
    for start in range(0, global_rows, batch_size):
        n = min(batch_size, global_rows - start)
        lo, hi = online_slice(start, n, rank, world)
        out.extend(range(lo, hi))
    return out
