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
"""

from __future__ import annotations

import ctypes as C

from . import _native

GELU, RELU, NONE = 2, 1, 0
OUT_BF16, OUT_F32, OUT_QKV = 0, 1, 2


class GemmEpilogue(C.Structure):
    _fields_ = [("bias", C.c_void_p), ("residual", C.c_void_p), ("ldr", C.c_int64),
                ("act", C.c_int32), ("out_mode", C.c_int32), ("seq_len", C.c_int32),
                ("heads", C.c_int32), ("tile_n", C.c_int32), ("rows_per_item", C.c_int32),
                ("count_dev", C.c_void_p)]


def gemm(lib, A, lda, W, D, ldd, M, N, K, stream, bias=None, residual=None, act=NONE,
         out_mode=OUT_BF16, seq_len=0, heads=0, tile_n=0, count=None, rows_per_item=1):
    ep = GemmEpilogue(None if bias is None else bias.data_ptr(),
                      None if residual is None else residual.data_ptr(),
                      0 if residual is None else residual.stride(0), act, out_mode, seq_len,
                      heads, tile_n, rows_per_item if count is not None else 0,
                      None if count is None else count.data_ptr())
    _native.check("gg_gemm", lib.gg_gemm(C.c_void_p(A), lda, _native.ptr(W), W.stride(0),
                                         C.c_void_p(D), ldd, M, N, K, C.byref(ep), stream))


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
        self.w_pre = bf(sd["pre_classifier.weight"])
        self.b_pre = f32(sd["pre_classifier.bias"])
        ncls = 32  # classifier rows padded to the GEMM's N granularity with zeros
        w_cls = torch.zeros((ncls, self.DIM), dtype=torch.float32)
        w_cls[: self.num_labels] = sd["classifier.weight"].float().cpu()
        b_cls = torch.zeros(ncls, dtype=torch.float32)
        b_cls[: self.num_labels] = sd["classifier.bias"].float().cpu()
        self.w_cls, self.b_cls = bf(w_cls), f32(b_cls)
        M = max_batch * seq_len
        z = dict(dtype=torch.bfloat16, device=self.device)
        self.x = torch.empty((M, self.DIM), **z)
        self.x1 = torch.empty((M, self.DIM), **z)
        self.h = torch.empty((M, self.DIM), **z)
        self.qkv = torch.empty(3 * M * self.DIM, **z)
        self.ctx = torch.empty((M, self.DIM), **z)
        self.ffn = torch.empty((M, self.FFN), **z)
        self.pooled = torch.empty((max_batch, self.DIM), **z)
        self.logits = torch.empty((max_batch, ncls), dtype=torch.float32, device=self.device)

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
        _native.check("gg_embed_layernorm", lib.gg_embed_layernorm(
            _native.ptr(input_ids), _native.ptr(self.word), _native.ptr(self.pos),
            _native.ptr(self.x), _native.ptr(self.emb_g), _native.ptr(self.emb_b), M, S, D,
            C.c_float(self.EPS), cnt, st))
        x, x1, h = self.x.data_ptr(), self.x1.data_ptr(), self.h.data_ptr()
        dyn = dict(count=count, rows_per_item=S)
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
        gemm(lib, x, S * D, self.w_pre, self.pooled.data_ptr(), D, B, D, D, st, bias=self.b_pre,
             act=RELU, tile_n=64, count=count, rows_per_item=1)
        gemm(lib, self.pooled.data_ptr(), D, self.w_cls, self.logits.data_ptr(),
             self.logits.stride(0), B, self.w_cls.shape[0], D, st, bias=self.b_cls,
             out_mode=OUT_F32, tile_n=64, count=count, rows_per_item=1)
        return self.logits[:B, : self.num_labels]


def random_model(seed: int = 0, num_labels: int = 2):
    """Seeded random-init DistilBERT-base classifier (no pretrained weights offline)."""
    import torch
    from transformers import DistilBertConfig, DistilBertForSequenceClassification

    torch.manual_seed(seed)
    m = DistilBertForSequenceClassification(DistilBertConfig(num_labels=num_labels))
    return m.eval()
