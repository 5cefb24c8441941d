"""DistilBERT-base sequence classifier forward on sm_100a (north star subsystem 2).

Architecture of transformers' DistilBertForSequenceClassification (dim 768,
12 heads, FFN 3072, 6 layers, exact-erf GELU, LayerNorm eps 1e-12, learned
positions, CLS -> pre_classifier -> ReLU -> classifier), evaluated with the
kernels of csrc/ through the forward C ABI (include/greengate_b200_forward.h):

  embeddings + LN          gg_embed_layernorm            (HBM-bound)
  fused QKV projection     gg_gemm  OUT_QKV_HEADS        (tcgen05, Q pre-scaled, V^T)
  self-attention           gg_attention                  (tcgen05 QK^T and PV, TMEM)
  out_lin + residual       gg_gemm  residual epilogue
  sa_layer_norm            gg_layernorm
  lin1 + GELU              gg_gemm  GELU epilogue
  lin2 + residual          gg_gemm  residual epilogue
  output_layer_norm        gg_layernorm
  CLS head                 gg_gemm (strided CLS rows, ReLU) -> gg_gemm (fp32 logits)

Weights are packed once from a transformers module (bf16 matrices, fp32
bias/LN vectors); PyTorch only owns the buffers.

LayerNorm folding (default when max_batch * seq_len >= 4096, the CTA-pair GEMM
path; GG_LN_UNFUSED=1 keeps the LayerNorm kernels): no LayerNorm kernel runs
inside the encoder.  The residual GEMMs (out_lin, lin2) write the RAW sum h and
per-row statistics partials of it; the next GEMM on the normalized rows
(QKV, lin1) multiplies raw h by W' = W diag(gamma) and corrects per row in its
epilogue, rstd (h W'^T) - rstd mean s_j + (b_j + beta W^T), and the residual
GEMM downstream adds LN(h) = (h - mean) rstd gamma + beta on the fly (gg_gemm_ln).
Only the 128 CLS rows before the head go through gg_layernorm.
"""

from __future__ import annotations

import ctypes as C
import os

from . import _native

GELU, RELU, NONE = 2, 1, 0
OUT_BF16, OUT_F32, OUT_QKV = 0, 1, 2


class GemmEpilogue(C.Structure):
    _fields_ = [("bias", C.c_void_p), ("residual", C.c_void_p), ("ldr", C.c_int64),
                ("act", C.c_int32), ("out_mode", C.c_int32), ("seq_len", C.c_int32),
                ("heads", C.c_int32), ("tile_n", C.c_int32), ("rows_per_item", C.c_int32),
                ("count_dev", C.c_void_p)]


class GgDep(C.Structure):
    """gg_dep (include/greengate_b200_forward.h): tile-level dependencies."""
    _fields_ = [("wait", C.c_void_p), ("need", C.c_int32), ("signal", C.c_void_p), ("go", C.c_void_p),
                ("tiles", C.c_void_p)]


class GemmLn(C.Structure):
    """gg_gemm_ln_params (include/greengate_b200_forward.h)."""
    _fields_ = [("a_stats", C.c_void_p), ("a_colsum", C.c_void_p), ("r_stats", C.c_void_p),
                ("r_gamma", C.c_void_p), ("r_beta", C.c_void_p), ("out_stats", C.c_void_p),
                ("ln_width", C.c_int32), ("eps", C.c_float)]


def gemm(lib, A, lda, W, D, ldd, M, N, K, stream, bias=None, residual=None, act=NONE,
         out_mode=OUT_BF16, seq_len=0, heads=0, tile_n=0, count=None, rows_per_item=1, ln=None,
         ldr=None, dep=None):
    res_ptr = None if residual is None else (residual if isinstance(residual, int)
                                             else residual.data_ptr())
    if residual is not None and ldr is None:
        ldr = residual.stride(0)
    ep = GemmEpilogue(None if bias is None else bias.data_ptr(), res_ptr,
                      0 if residual is None else ldr, act, out_mode, seq_len,
                      heads, tile_n, rows_per_item if count is not None else 0,
                      None if count is None else count.data_ptr())
    if dep is not None:
        _native.check("gg_gemm_dep", lib.gg_gemm_dep(
            C.c_void_p(A), lda, _native.ptr(W), W.stride(0), C.c_void_p(D), ldd, M, N, K,
            C.byref(ep), None if ln is None else C.byref(ln), C.byref(dep), stream))
    elif ln is None:
        _native.check("gg_gemm", lib.gg_gemm(C.c_void_p(A), lda, _native.ptr(W), W.stride(0),
                                             C.c_void_p(D), ldd, M, N, K, C.byref(ep), stream))
    else:
        _native.check("gg_gemm_ln", lib.gg_gemm_ln(C.c_void_p(A), lda, _native.ptr(W), W.stride(0),
                                                   C.c_void_p(D), ldd, M, N, K, C.byref(ep),
                                                   C.byref(ln), stream))


class DistilBertB200:
    """Packed weights + activation buffers for up to `max_batch` sequences of `seq_len`."""

    DIM, HEADS, FFN, EPS = 768, 12, 3072, 1e-12

    def __init__(self, hf_model, max_batch: int = 128, seq_len: int = 128, device="cuda"):
        torch = _native.require_cuda()
        self.lib = _native.load()
        # stream-K workspace now, before any CUDA graph capture of the forward
        _native.check("gg_streamk_reserve", self.lib.gg_streamk_reserve())
        self.device = torch.device(device)
        self.max_batch, self.seq_len = max_batch, seq_len
        cfg = hf_model.config
        assert cfg.dim == self.DIM and cfg.n_heads == self.HEADS and cfg.hidden_dim == self.FFN
        assert cfg.activation == "gelu" and seq_len == 128
        self.num_labels = cfg.num_labels
        sd = {k: v.detach() for k, v in hf_model.state_dict().items()}

        def bf(t):
            return t.to(device=self.device, dtype=torch.bfloat16).contiguous()

        def f32(t):
            return t.to(device=self.device, dtype=torch.float32).contiguous()

        p = "distilbert."
        self.word = bf(sd[p + "embeddings.word_embeddings.weight"])
        self.pos = bf(sd[p + "embeddings.position_embeddings.weight"])
        self.emb_g = f32(sd[p + "embeddings.LayerNorm.weight"])
        self.emb_b = f32(sd[p + "embeddings.LayerNorm.bias"])
        self.layers = []
        for i in range(cfg.n_layers):
            q = f"{p}transformer.layer.{i}."
            a = q + "attention."
            self.layers.append(dict(
                w_qkv=bf(torch.cat([sd[a + "q_lin.weight"], sd[a + "k_lin.weight"], sd[a + "v_lin.weight"]])),
                b_qkv=f32(torch.cat([sd[a + "q_lin.bias"], sd[a + "k_lin.bias"], sd[a + "v_lin.bias"]])),
                w_o=bf(sd[a + "out_lin.weight"]), b_o=f32(sd[a + "out_lin.bias"]),
                ln1_g=f32(sd[q + "sa_layer_norm.weight"]), ln1_b=f32(sd[q + "sa_layer_norm.bias"]),
                w1=bf(sd[q + "ffn.lin1.weight"]), b1=f32(sd[q + "ffn.lin1.bias"]),
                w2=bf(sd[q + "ffn.lin2.weight"]), b2=f32(sd[q + "ffn.lin2.bias"]),
                ln2_g=f32(sd[q + "output_layer_norm.weight"]), ln2_b=f32(sd[q + "output_layer_norm.bias"]),
            ))
        M = max_batch * seq_len
        self.fused_ln = M >= 4096 and os.environ.get("GG_LN_UNFUSED") != "1"
        if self.fused_ln:
            self._fold_layernorms(sd)
        self.w_pre = bf(sd["pre_classifier.weight"])
        self.b_pre = f32(sd["pre_classifier.bias"])
        ncls = 32  # classifier rows padded to the GEMM's N granularity with zeros
        w_cls = torch.zeros((ncls, self.DIM), dtype=torch.float32)
        w_cls[: self.num_labels] = sd["classifier.weight"].float().cpu()
        b_cls = torch.zeros(ncls, dtype=torch.float32)
        b_cls[: self.num_labels] = sd["classifier.bias"].float().cpu()
        self.w_cls, self.b_cls = bf(w_cls), f32(b_cls)
        z = dict(dtype=torch.bfloat16, device=self.device)
        self.x = torch.empty((M, self.DIM), **z)
        self.x1 = torch.empty((M, self.DIM), **z)
        self.h = torch.empty((M, self.DIM), **z)
        self.qkv = torch.empty(3 * M * self.DIM, **z)
        self.ctx = torch.empty((M, self.DIM), **z)
        self.ffn = torch.empty((M, self.FFN), **z)
        self.pooled = torch.empty((max_batch, self.DIM), **z)
        self.cls = torch.empty((max_batch, self.DIM), **z)
        self.logits = torch.empty((max_batch, ncls), dtype=torch.float32, device=self.device)
        # LayerNorm folding: per-row statistics partials of h1 / h2 ([768 / 128][M] float2)
        parts = self.DIM // 128
        self.st1 = torch.empty((parts, M, 2), dtype=torch.float32, device=self.device)
        self.st2 = torch.empty((parts, M, 2), dtype=torch.float32, device=self.device)
        # tile-level dependencies between the encoder's kernels (gg_dep; folded path):
        # [go | per layer: QKV, attention, out_lin, lin1, lin2 counters per sequence |
        #  per layer and kernel: dynamic tile counter]
        # Opt-in (GG_DEP=1): measured no faster than grid-wide PDL waits on B200 --
        # the row-block raster and per-tile signalling cost the QKV / lin1 epilogues
        # about what the overlap of kernel tails recovers.
        self.use_deps = self.fused_ln and os.environ.get("GG_DEP") == "1"
        self.dyn_tiles = os.environ.get("GG_STATIC_TILES") != "1"
        nl = len(self.layers)
        self.deps = torch.zeros(1 + nl * 5 * max_batch + nl * 5, dtype=torch.int32,
                                device=self.device)
        # fused feed-forward block (gg_ffn_pair, opt-in GG_FFN_FUSE=1): per layer, lin1
        # tiles published per 128-row unit + the tile claim counter; zeroed once per
        # forward.  Bit-identical to the two launches but measured no faster (DESIGN.md
        # section 7, finding H): the merged queue's last lin2 tiles leave the same
        # imbalance as FFN-down's partial wave, and the row-block raster slows lin1.
        self.use_ffn_fused = self.fused_ln and os.environ.get("GG_FFN_FUSE") == "1"
        self.ffn_units = max_batch * seq_len // 128
        self.ffn_ctr = torch.zeros(nl * (self.ffn_units + 1), dtype=torch.int32, device=self.device)
        # classification head as one launch (gg_cls_head): column-block partials of the
        # classifier + per-16-row arrival counters (re-zeroed by the kernel)
        self.fused_head = os.environ.get("GG_HEAD_UNFUSED") != "1"
        hb = int(self.lib.gg_cls_head_scratch_bytes(max_batch))
        self.head_part = torch.empty(hb // 4, dtype=torch.float32, device=self.device)
        self.head_arr = torch.zeros((max_batch + 15) // 16, dtype=torch.int32, device=self.device)

    def _fold_layernorms(self, sd) -> None:
        """W' = W diag(gamma) (bf16), s_j = sum_k W'_jk and c_j = b_j + sum_k beta_k W_jk
        for every GEMM that consumes a LayerNorm output as its A operand: QKV of
        layer L >= 1 (output_layer_norm of L - 1), lin1 of every layer
        (sa_layer_norm).  fp64 on the host, once."""
        torch = _native.require_cuda()

        def fold(w_fp32, b, gamma, beta):
            w = w_fp32.double().cpu()
            g, bt = gamma.double().cpu(), beta.double().cpu()
            wp = (w * g[None, :]).to(torch.bfloat16)
            colsum = wp.double().sum(dim=1)
            c = b.double().cpu() + w @ bt
            dev = self.device
            return (wp.to(dev).contiguous(), colsum.float().to(dev).contiguous(),
                    c.float().to(dev).contiguous())
        p = "distilbert.transformer.layer."
        for i, L in enumerate(self.layers):
            a = f"{p}{i}.attention."
            if i > 0:
                P = self.layers[i - 1]
                w_qkv = torch.cat([sd[a + "q_lin.weight"], sd[a + "k_lin.weight"],
                                   sd[a + "v_lin.weight"]])
                L["w_qkv_f"], L["s_qkv"], L["c_qkv"] = fold(w_qkv, L["b_qkv"], P["ln2_g"],
                                                            P["ln2_b"])
            L["w1_f"], L["s_1"], L["c_1"] = fold(sd[f"{p}{i}.ffn.lin1.weight"], L["b1"],
                                                 L["ln1_g"], L["ln1_b"])

    def flops(self, batch: int) -> float:
        """Algorithmic FLOPs of one forward (11.17 GF/seq at S=128)."""
        S, D, F, L = self.seq_len, self.DIM, self.FFN, len(self.layers)
        M = batch * S
        lin = 2 * M * D * (3 * D + D + F + F)
        attn = 2 * 2 * batch * self.HEADS * S * S * (D // self.HEADS)
        head = 2 * batch * D * (D + self.num_labels)
        return float(L * (lin + attn) + head)

    def forward(self, input_ids, attention_mask=None, batch: int | None = None, stream=None,
                count=None):
        """input_ids: CUDA int32 [B, S]; attention_mask: CUDA int32 [B, S] or None.
        count: optional CUDA int32 [1] = number of valid sequences (dynamic batch,
        read on the device).  Returns fp32 logits [B, num_labels] (a view)."""
        lib = self.lib
        B = int(input_ids.shape[0]) if batch is None else int(batch)
        S, D = self.seq_len, self.DIM
        assert B <= self.max_batch and input_ids.dtype.itemsize == 4
        M = B * S
        st = _native.stream_ptr(stream)
        cnt = _native.ptr(count)
        self._mask = attention_mask
        _native.check("gg_embed_layernorm", lib.gg_embed_layernorm(
            _native.ptr(input_ids), _native.ptr(self.word), _native.ptr(self.pos),
            _native.ptr(self.x), _native.ptr(self.emb_g), _native.ptr(self.emb_b), M, S, D,
            C.c_float(self.EPS), cnt, st))
        x, x1, h = self.x.data_ptr(), self.x1.data_ptr(), self.h.data_ptr()
        dyn = dict(count=count, rows_per_item=S)
        if self.fused_ln:
            return self._forward_folded(B, S, D, M, st, cnt, count, dyn)
        for L in self.layers:
            gemm(lib, x, D, L["w_qkv"], self.qkv.data_ptr(), 3 * D, M, 3 * D, D, st,
                 bias=L["b_qkv"], out_mode=OUT_QKV, seq_len=S, heads=self.HEADS, **dyn)
            _native.check("gg_attention", lib.gg_attention(
                _native.ptr(self.qkv), _native.ptr(attention_mask), _native.ptr(self.ctx), D, B,
                self.HEADS, S, cnt, st))
            gemm(lib, self.ctx.data_ptr(), D, L["w_o"], h, D, M, D, D, st, bias=L["b_o"],
                 residual=self.x, **dyn)
            _native.check("gg_layernorm", lib.gg_layernorm(
                C.c_void_p(h), D, C.c_void_p(x1), D, _native.ptr(L["ln1_g"]),
                _native.ptr(L["ln1_b"]), M, D, C.c_float(self.EPS), cnt, S, st))
            gemm(lib, x1, D, L["w1"], self.ffn.data_ptr(), self.FFN, M, self.FFN, D, st,
                 bias=L["b1"], act=GELU, **dyn)
            gemm(lib, self.ffn.data_ptr(), self.FFN, L["w2"], h, D, M, D, self.FFN, st,
                 bias=L["b2"], residual=self.x1, **dyn)
            _native.check("gg_layernorm", lib.gg_layernorm(
                C.c_void_p(h), D, C.c_void_p(x), D, _native.ptr(L["ln2_g"]),
                _native.ptr(L["ln2_b"]), M, D, C.c_float(self.EPS), cnt, S, st))
        # CLS rows (stride S*D) -> pre_classifier + ReLU -> classifier (fp32 logits)
        if self.fused_head:
            return self._head(x, S * D, None, B, st, cnt)
        gemm(lib, x, S * D, self.w_pre, self.pooled.data_ptr(), D, B, D, D, st, bias=self.b_pre,
             act=RELU, tile_n=64, count=count, rows_per_item=1)
        gemm(lib, self.pooled.data_ptr(), D, self.w_cls, self.logits.data_ptr(),
             self.logits.stride(0), B, self.w_cls.shape[0], D, st, bias=self.b_cls,
             out_mode=OUT_F32, tile_n=64, count=count, rows_per_item=1)
        return self.logits[:B, : self.num_labels]


    def _forward_folded(self, B, S, D, M, st, cnt, count, dyn):
        """Encoder with every LayerNorm folded into the GEMMs (class docstring)."""
        lib, eps = self.lib, self.EPS
        # Tile-level dependencies: each kernel of the encoder waits per sequence for
        # the tiles it reads instead of the whole previous grid, so a kernel's first
        # tiles start on the SMs its predecessor's last wave leaves idle.
        dp = self.deps.data_ptr()
        nl, mb = len(self.layers), self.max_batch
        go = C.c_void_p(dp)

        def ctr(i, k):   # k: 0 QKV, 1 attention, 2 out_lin, 3 lin1, 4 lin2
            return C.c_void_p(dp + 4 * (1 + (i * 5 + k) * mb))

        def dep(i, k, wait, need):
            if not self.use_deps:
                return None
            sig = ctr(i, k) if not (i == nl - 1 and k == 4) else None
            tiles = C.c_void_p(dp + 4 * (1 + nl * 5 * mb + i * 5 + k)) if self.dyn_tiles else None
            return GgDep(wait, need, sig, go, tiles)
        if self.use_deps:
            _native.check("gg_zero_async", lib.gg_zero_async(_native.ptr(self.deps),
                                                             self.deps.numel() * 4, st))
        if self.use_ffn_fused:
            _native.check("gg_zero_async", lib.gg_zero_async(_native.ptr(self.ffn_ctr),
                                                             self.ffn_ctr.numel() * 4, st))
        H = self.HEADS
        x0 = self.x.data_ptr()       # embeddings + LayerNorm (normalized)
        hA = self.x1.data_ptr()      # h1 = ctx W_o^T + b_o + x   (raw, LN1 folded downstream)
        hB = self.h.data_ptr()       # h2 = ffn W_2^T + b_2 + x1  (raw, LN2 folded downstream)
        p1, p2 = self.st1.data_ptr(), self.st2.data_ptr()
        f = C.c_float(eps)
        for i, L in enumerate(self.layers):
            P = self.layers[i - 1] if i > 0 else None
            # QKV waits for the previous layer's lin2 (3 column tiles per sequence)
            d_qkv = dep(i, 0, None if i == 0 else ctr(i - 1, 4), 3)
            if i == 0:
                gemm(lib, x0, D, L["w_qkv"], self.qkv.data_ptr(), 3 * D, M, 3 * D, D, st,
                     bias=L["b_qkv"], out_mode=OUT_QKV, seq_len=S, heads=H, dep=d_qkv, **dyn)
            else:
                gemm(lib, hB, D, L["w_qkv_f"], self.qkv.data_ptr(), 3 * D, M, 3 * D, D, st,
                     bias=L["c_qkv"], out_mode=OUT_QKV, seq_len=S, heads=H,
                     ln=GemmLn(p2, L["s_qkv"].data_ptr(), None, None, None, None, D, f),
                     dep=d_qkv, **dyn)
            d_att = dep(i, 1, ctr(i, 0), 3 * D // 256)
            if d_att is None:
                _native.check("gg_attention", lib.gg_attention(
                    _native.ptr(self.qkv), _native.ptr(self._mask), _native.ptr(self.ctx), D, B,
                    H, S, cnt, st))
            else:
                _native.check("gg_attention_dep", lib.gg_attention_dep(
                    _native.ptr(self.qkv), _native.ptr(self._mask), _native.ptr(self.ctx), D, B,
                    H, S, cnt, C.byref(d_att), st))
            d_out = dep(i, 2, ctr(i, 1), H)
            if i == 0:   # residual = x0 (already normalized)
                gemm(lib, self.ctx.data_ptr(), D, L["w_o"], hA, D, M, D, D, st, bias=L["b_o"],
                     residual=x0, ldr=D,
                     ln=GemmLn(None, None, None, None, None, p1, D, f), dep=d_out, **dyn)
            else:        # residual = LN2_{i-1}(h2)
                gemm(lib, self.ctx.data_ptr(), D, L["w_o"], hA, D, M, D, D, st, bias=L["b_o"],
                     residual=hB, ldr=D,
                     ln=GemmLn(None, None, p2, P["ln2_g"].data_ptr(), P["ln2_b"].data_ptr(), p1,
                               D, f), dep=d_out, **dyn)
            if self.use_ffn_fused and not self.use_deps:
                # lin1 + GELU and lin2 + residual as one persistent kernel (tile queue)
                u = self.ffn_units + 1
                cbase = self.ffn_ctr.data_ptr() + 4 * i * u
                _native.check("gg_ffn_pair", lib.gg_ffn_pair(
                    C.c_void_p(hA), _native.ptr(L["w1_f"]), _native.ptr(self.ffn), _native.ptr(L["w2"]),
                    C.c_void_p(hB), M, D, self.FFN, cnt, S if count is not None else 0,
                    _native.ptr(L["c_1"]), _native.ptr(L["s_1"]), C.c_void_p(p1), _native.ptr(L["b2"]),
                    C.c_void_p(p1), _native.ptr(L["ln1_g"]), _native.ptr(L["ln1_b"]), C.c_void_p(p2), f,
                    C.c_void_p(cbase), C.c_void_p(cbase + 4 * self.ffn_units), st))
            else:
                gemm(lib, hA, D, L["w1_f"], self.ffn.data_ptr(), self.FFN, M, self.FFN, D, st,
                     bias=L["c_1"], act=GELU,
                     ln=GemmLn(p1, L["s_1"].data_ptr(), None, None, None, None, D, f),
                     dep=dep(i, 3, ctr(i, 2), D // 256), **dyn)
                gemm(lib, self.ffn.data_ptr(), self.FFN, L["w2"], hB, D, M, D, self.FFN, st,
                     bias=L["b2"], residual=hA, ldr=D,
                     ln=GemmLn(None, None, p1, L["ln1_g"].data_ptr(), L["ln1_b"].data_ptr(), p2, D, f),
                     dep=dep(i, 4, ctr(i, 3), self.FFN // 256), **dyn)
        last = self.layers[-1]
        if self.fused_head:
            return self._head(hB, S * D, last, B, st, cnt)
        # the head reads only the CLS rows: LayerNorm of those B rows (stride S*D)
        _native.check("gg_layernorm", lib.gg_layernorm(
            C.c_void_p(hB), S * D, _native.ptr(self.cls), D, _native.ptr(last["ln2_g"]),
            _native.ptr(last["ln2_b"]), B, D, f, cnt, 1, st))
        gemm(lib, self.cls.data_ptr(), D, self.w_pre, self.pooled.data_ptr(), D, B, D, D, st,
             bias=self.b_pre, act=RELU, tile_n=64, count=count, rows_per_item=1)
        gemm(lib, self.pooled.data_ptr(), D, self.w_cls, self.logits.data_ptr(),
             self.logits.stride(0), B, self.w_cls.shape[0], D, st, bias=self.b_cls,
             out_mode=OUT_F32, tile_n=64, count=count, rows_per_item=1)
        return self.logits[:B, : self.num_labels]

    def _head(self, rows_ptr, ld, ln, B, st, cnt):
        """LayerNorm (ln = the last layer's output_layer_norm, or None when the rows are
        already normalized) + pre_classifier + ReLU + classifier on the B CLS rows in
        one launch (gg_cls_head)."""
        _native.check("gg_cls_head", self.lib.gg_cls_head(
            C.c_void_p(rows_ptr), ld, _native.ptr(ln["ln2_g"]) if ln else None,
            _native.ptr(ln["ln2_b"]) if ln else None, C.c_float(self.EPS), _native.ptr(self.w_pre),
            _native.ptr(self.b_pre), _native.ptr(self.w_cls), _native.ptr(self.b_cls),
            self.num_labels, _native.ptr(self.logits), self.logits.stride(0), B, self.max_batch,
            cnt, _native.ptr(self.head_part), _native.ptr(self.head_arr), st))
        return self.logits[:B, : self.num_labels]


def random_model(seed: int = 0, num_labels: int = 2):
    """Seeded random-init DistilBERT-base classifier (no pretrained weights offline)."""
    import torch
    from transformers import DistilBertConfig, DistilBertForSequenceClassification

    torch.manual_seed(seed)
    m = DistilBertForSequenceClassification(DistilBertConfig(num_labels=num_labels))
    return m.eval()
