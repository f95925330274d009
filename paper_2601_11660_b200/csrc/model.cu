// Whole-network runner: the native replacement of graph.forward's
// interpreter loop (graph.py:413-458).
//
// Planning resolves every layer's output to a view (buffer, pixel stride,
// word offset) inside one caller-provided workspace. Concatenation
// (layers.py:369-384) is resolved at plan time into a split view: both
// operands keep their own contiguous tensors and the consuming conv reads
// words [0, wpp_a) of a pixel from the first and the rest from the second
// (conv_tc: one TMA tensor map per operand). A concat step launches nothing,
// the skip tensor is never copied, and no kernel writes part of a 32-B
// sector that another kernel fills (the half-sector read-modify-write an
// interleaved concat buffer costs at DRAM). The forward
// then enqueues one kernel per conv / pool step on the caller's stream, which
// the Python host captures into a CUDA graph.
#include <cuda_runtime.h>

#include <string>
#include <vector>

#include "common.cuh"

using namespace mbu;

namespace {

struct Layer {
  int type = 0;
  mbu_conv *conv = nullptr;
  mbu_fconv *fconv = nullptr;
  int apply_sign = 0;
  int skip = -1;
  // planned
  int src = -1;          // producer of this layer's input (-1 = image)
  int n = 0, h = 0, w = 0;
  int out_kind = 0;      // 0 packed bits, 1 float64 (logits)
  int wpp = 0;           // bits: words per pixel; float: channels
  int buf = -1, stride = 0, offset = 0;  // (concat: no buffer, a split view of src + skip)
  int acc_buf = -1, acc_c = 0, acc_f64 = 0;
};

}  // namespace

struct mbu_model {
  int device = 0;
  std::vector<Layer> layers;
  int planned = 0, n = 0, H = 0, W = 0, trace = 0, in_c = 0;
  std::vector<size_t> buf_off, buf_bytes;
  size_t ws = 0;
  // optional per-layer CUDA-event timing (bench.py roofline)
  int timing = 0;
  std::vector<cudaEvent_t> events;  // layers + 1
};

static int add_buf(mbu_model *m, size_t bytes) {
  const size_t align = 256;
  size_t off = (m->ws + align - 1) / align * align;
  m->buf_off.push_back(off);
  m->buf_bytes.push_back(bytes);
  m->ws = off + bytes;
  return int(m->buf_off.size()) - 1;
}

extern "C" {

int mbu_model_create(mbu_model **out, int device) {
  *out = new mbu_model();
  (*out)->device = device;
  return MBU_OK;
}

int mbu_model_destroy(mbu_model *m) {
  if (!m) return MBU_OK;
  for (auto e : m->events) cudaEventDestroy(e);
  for (auto &l : m->layers) {
    mbu_conv_destroy(l.conv);
    mbu_fconv_destroy(l.fconv);
  }
  delete m;
  return MBU_OK;
}

int mbu_model_add_conv(mbu_model *m, mbu_conv *conv) {
  Layer l;
  l.type = conv->transposed ? MBU_LAYER_BIT_TCONV : MBU_LAYER_BIT_CONV;
  l.conv = conv;
  m->layers.push_back(l);
  m->planned = 0;
  return MBU_OK;
}

int mbu_model_add_fconv(mbu_model *m, mbu_fconv *conv, int apply_sign) {
  Layer l;
  l.type = MBU_LAYER_FLOAT_CONV;
  l.fconv = conv;
  l.apply_sign = apply_sign;
  m->layers.push_back(l);
  m->planned = 0;
  return MBU_OK;
}

int mbu_model_add_maxpool(mbu_model *m) {
  Layer l;
  l.type = MBU_LAYER_MAXPOOL;
  m->layers.push_back(l);
  m->planned = 0;
  return MBU_OK;
}

int mbu_model_add_concat(mbu_model *m, int skip) {
  if (skip < 0 || skip >= int(m->layers.size()))
    return fail(MBU_ERR_ENGINE, "concat skip index out of range");
  Layer l;
  l.type = MBU_LAYER_CONCAT;
  l.skip = skip;
  m->layers.push_back(l);
  m->planned = 0;
  return MBU_OK;
}

int mbu_model_plan(mbu_model *m, int n, int H, int W, int trace, size_t *ws_bytes) {
  auto &L = m->layers;
  if (L.empty() || L[0].type != MBU_LAYER_FLOAT_CONV || L[0].fconv->bits_input)
    return fail(MBU_ERR_UNSUPPORTED, "the first layer must be a float conv on the image");
  m->planned = 0;
  m->n = n; m->H = H; m->W = W; m->trace = trace;
  m->in_c = L[0].fconv->c_in;
  m->buf_off.clear();
  m->buf_bytes.clear();
  m->ws = 0;
  // ---- shapes
  int cn = n, ch = H, cw = W, ckind = 1, cwpp = m->in_c;
  for (int i = 0; i < int(L.size()); ++i) {
    Layer &l = L[i];
    l.src = i - 1;
    l.buf = -1;
    l.acc_buf = -1;
    if (l.type == MBU_LAYER_FLOAT_CONV) {
      const mbu_fconv *f = l.fconv;
      if ((ckind == 0) != bool(f->bits_input))
        return fail(MBU_ERR_LAYOUT, "float conv input kind mismatch at layer " + std::to_string(i));
      if (ckind == 1 && cwpp != f->c_in) return fail(MBU_ERR_SHAPE, "float conv c_in mismatch");
      l.n = cn;
      l.h = (ch + 2 * f->pad - f->kh) / f->stride + 1;
      l.w = (cw + 2 * f->pad - f->kw) / f->stride + 1;
      if (l.apply_sign) {
        l.out_kind = 0;
        l.wpp = ((f->c_out + 127) / 128) * 2;
      } else {
        l.out_kind = 1;
        l.wpp = f->c_out;
        if (i != int(L.size()) - 1)
          return fail(MBU_ERR_UNSUPPORTED, "a float output is only supported as the last layer");
      }
      if (trace && l.apply_sign) { l.acc_c = f->c_out; l.acc_f64 = 1; }
    } else if (l.type == MBU_LAYER_BIT_CONV || l.type == MBU_LAYER_BIT_TCONV) {
      const mbu_conv *c = l.conv;
      if (ckind != 0) return fail(MBU_ERR_LAYOUT, "bit conv needs a packed input");
      if (cwpp != c->wpp) return fail(MBU_ERR_LAYOUT, "bit conv input words-per-pixel mismatch at layer " + std::to_string(i));
      l.n = cn;
      if (c->transposed) { l.h = ch * c->stride; l.w = cw * c->stride; }
      else {
        l.h = (ch + 2 * c->pad - c->kh) / c->stride + 1;
        l.w = (cw + 2 * c->pad - c->kw) / c->stride + 1;
      }
      if (l.h <= 0 || l.w <= 0) return fail(MBU_ERR_SHAPE, "kernel larger than padded input");
      l.out_kind = 0;
      l.wpp = c->out_wpp;
      if (!c->has_threshold) return fail(MBU_ERR_ENGINE, "model conv without thresholds");
      if (trace) { l.acc_c = c->c_out; l.acc_f64 = 0; }
    } else if (l.type == MBU_LAYER_MAXPOOL) {
      if (ckind != 0) return fail(MBU_ERR_LAYOUT, "maxpool needs a packed input");
      if (ch % 2 || cw % 2) return fail(MBU_ERR_SHAPE, "maxpool extents must be even");
      l.n = cn; l.h = ch / 2; l.w = cw / 2; l.out_kind = 0; l.wpp = cwpp;
    } else {  // concat
      const Layer &b = L[l.skip];
      if (ckind != 0 || b.out_kind != 0) return fail(MBU_ERR_LAYOUT, "concat needs packed operands");
      if (b.n != cn || b.h != ch || b.w != cw) return fail(MBU_ERR_SHAPE, "concat spatial extents differ");
      l.n = cn; l.h = ch; l.w = cw; l.out_kind = 0; l.wpp = cwpp + b.wpp;
    }
    cn = l.n; ch = l.h; cw = l.w; ckind = l.out_kind; cwpp = l.wpp;
  }
  // ---- concat operands: plain tensors; only bit convs read a concat
  for (int i = 0; i < int(L.size()); ++i) {
    if (L[i].type != MBU_LAYER_CONCAT) continue;
    for (int opnd : {L[i].src, L[i].skip})
      if (opnd < 0 || L[opnd].type == MBU_LAYER_CONCAT)
        return fail(MBU_ERR_UNSUPPORTED, "concat of a concat is not supported");
    for (int j = i + 1; j < int(L.size()); ++j)
      if ((L[j].src == i || (L[j].type == MBU_LAYER_CONCAT && L[j].skip == i)) &&
          L[j].type != MBU_LAYER_BIT_CONV && L[j].type != MBU_LAYER_BIT_TCONV)
        return fail(MBU_ERR_UNSUPPORTED, "a concat must feed a bit conv");
  }
  // ---- buffers
  for (int i = 0; i < int(L.size()); ++i) {
    Layer &l = L[i];
    if (l.out_kind == 0 && l.type != MBU_LAYER_CONCAT) {
      l.buf = add_buf(m, size_t(l.n) * l.h * l.w * l.wpp * 8);
      l.stride = l.wpp;
      l.offset = 0;
    }
    if (l.acc_c) l.acc_buf = add_buf(m, size_t(l.n) * l.h * l.w * l.acc_c * (l.acc_f64 ? 8 : 4));
  }
  m->planned = 1;
  *ws_bytes = m->ws;
  return MBU_OK;
}

int mbu_forward(mbu_model *m, const double *image, double *logits, uint8_t *mask, void *ws,
                size_t ws_bytes, int path, void *stream) {
  if (!m->planned) return fail(MBU_ERR_ENGINE, "mbu_forward before mbu_model_plan");
  if (ws_bytes < m->ws) return fail(MBU_ERR_ENGINE, "workspace too small");
  if (!logits) return fail(MBU_ERR_ENGINE, "logits buffer required");
  cudaStream_t st = as_stream(stream);
  char *base = static_cast<char *>(ws);
  auto view_of = [&](int i) -> ActView {
    const Layer &l = m->layers[i];
    if (l.type == MBU_LAYER_CONCAT) {  // split view: src words, then the skip's
      const Layer &a = m->layers[l.src], &b = m->layers[l.skip];
      return ActView{reinterpret_cast<const uint64_t *>(base + m->buf_off[a.buf]), l.n, l.h, l.w, l.wpp,
                     a.stride, a.offset, reinterpret_cast<const uint64_t *>(base + m->buf_off[b.buf]),
                     b.stride, a.wpp};
    }
    return ActView{reinterpret_cast<const uint64_t *>(base + m->buf_off[l.buf]), l.n, l.h, l.w,
                   l.wpp, l.stride, l.offset, nullptr, 0, 0};
  };
  const bool timed = m->timing && int(m->events.size()) == int(m->layers.size()) + 1;
  // MBU_OPT_FUSED_HEAD: the final 1x1 head folds into the epilogue of the bit
  // conv right before it when that conv's output feeds nothing else and is not traced
  auto head_after = [&](int i) -> const mbu_fconv * {
    const int nl = int(m->layers.size());
    if (!g_fused_head || g_force_generic_fconv || i + 1 >= nl) return nullptr;
    const Layer &c = m->layers[i], &h = m->layers[i + 1];
    if (c.type != MBU_LAYER_BIT_CONV || c.acc_buf >= 0 || h.type != MBU_LAYER_FLOAT_CONV || h.apply_sign ||
        h.src != i)
      return nullptr;
    for (int j = 0; j < nl; ++j)
      if (j != i + 1 && (m->layers[j].src == i || (m->layers[j].type == MBU_LAYER_CONCAT && m->layers[j].skip == i)))
        return nullptr;
    const mbu_fconv *f = h.fconv;
    if (!f->d_head_nib || !f->bits_input || f->c_out != 1 || f->c_in != 64 || f->kh != 1 || f->kw != 1 ||
        f->stride != 1 || f->pad != 0)
      return nullptr;
    return f;
  };
  int fused_head = -1;
  for (int i = 0; i < int(m->layers.size()); ++i) {
    const Layer &l = m->layers[i];
    if (timed) MBU_TRY(check_cuda(cudaEventRecord(m->events[i], st), "cudaEventRecord"));
    if (i == fused_head) continue;
    uint64_t *out = l.buf >= 0 ? reinterpret_cast<uint64_t *>(base + m->buf_off[l.buf]) : nullptr;
    void *acc = l.acc_buf >= 0 ? base + m->buf_off[l.acc_buf] : nullptr;
    int in_h = l.src < 0 ? m->H : m->layers[l.src].h;
    int in_w = l.src < 0 ? m->W : m->layers[l.src].w;
    switch (l.type) {
      case MBU_LAYER_FLOAT_CONV: {
        ActView xb{};
        if (l.src >= 0) xb = view_of(l.src);
        if (l.apply_sign)
          MBU_TRY(launch_fconv(l.fconv, l.src < 0 ? image : nullptr, xb, m->n, in_h, in_w,
                               static_cast<double *>(acc), out, l.stride, l.offset, nullptr, st));
        else
          MBU_TRY(launch_fconv(l.fconv, l.src < 0 ? image : nullptr, xb, m->n, in_h, in_w,
                               logits, nullptr, 0, 0, mask, st));
        break;
      }
      case MBU_LAYER_BIT_CONV:
      case MBU_LAYER_BIT_TCONV: {
        const mbu_fconv *hf = head_after(i);
        HeadFuse fuse{hf ? hf->d_head_nib : nullptr, hf ? hf->d_bias : nullptr, logits, mask, false};
        MBU_TRY(conv_run(l.conv, view_of(l.src), static_cast<int32_t *>(acc), out, l.stride,
                         l.offset, path, st, hf ? &fuse : nullptr));
        if (fuse.done) fused_head = i + 1;
        break;
      }
      case MBU_LAYER_MAXPOOL:
        MBU_TRY(launch_maxpool(view_of(l.src), out, l.stride, l.offset, st));
        break;
      default:
        break;  // concat: resolved at plan time
    }
  }
  if (timed) MBU_TRY(check_cuda(cudaEventRecord(m->events.back(), st), "cudaEventRecord"));
  return MBU_OK;
}

int mbu_model_set_timing(mbu_model *m, int enable) {
  if (enable && m->events.size() != m->layers.size() + 1) {
    for (auto e : m->events) cudaEventDestroy(e);
    m->events.assign(m->layers.size() + 1, nullptr);
    for (auto &e : m->events) MBU_TRY(check_cuda(cudaEventCreate(&e), "cudaEventCreate"));
  }
  m->timing = enable;
  return MBU_OK;
}

int mbu_model_layer_times(mbu_model *m, float *ms_out) {
  if (m->events.size() != m->layers.size() + 1) return fail(MBU_ERR_ENGINE, "timing not enabled");
  MBU_TRY(check_cuda(cudaEventSynchronize(m->events.back()), "cudaEventSynchronize"));
  for (size_t i = 0; i + 1 < m->events.size(); ++i)
    MBU_TRY(check_cuda(cudaEventElapsedTime(&ms_out[i], m->events[i], m->events[i + 1]), "cudaEventElapsedTime"));
  return MBU_OK;
}

int mbu_model_layer_info(mbu_model *m, int i, int *out_kind, int *n, int *h, int *w,
                         int *channels_or_wpp, int *pixel_stride, int *word_offset,
                         size_t *out_byte_offset, size_t *acc_byte_offset, int *acc_channels) {
  if (!m->planned) return fail(MBU_ERR_ENGINE, "model not planned");
  if (i < 0 || i >= int(m->layers.size())) return fail(MBU_ERR_ENGINE, "layer index out of range");
  const Layer &l = m->layers[i];
  *out_kind = l.out_kind;
  *n = l.n; *h = l.h; *w = l.w;
  *channels_or_wpp = l.wpp;
  *pixel_stride = l.stride;
  *word_offset = l.offset;
  *out_byte_offset = l.buf >= 0 ? m->buf_off[l.buf] : size_t(-1);
  *acc_byte_offset = l.acc_buf >= 0 ? m->buf_off[l.acc_buf] : size_t(-1);
  *acc_channels = l.acc_c;
  return MBU_OK;
}

}  // extern "C"
