/*
 * vc_oracle.h -- CPU restatement of the VeriCache decode-loop path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product library links, loads or
 * calls this code; it is the checker that tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline leg compare the CUDA path against.
 *
 * Parity pinning:
 *   - accept / protocol / drop-index generation restate the reference
 *     (/root/reference/proj/src/specloop.cpp:37-92, compressor.cpp:114-171)
 *     and are pinned bit-for-bit against the compiled reference (oracle/_ref)
 *     and the golden vectors of proj/tests/test_specloop.cpp:86-115,
 *     test_compressor.cpp:43-165.
 *   - quantisation codes, attention, the model forward and top-k selection
 *     have NO numeric reference in /root/reference:
 *     for those rows the parity is "unpinned by the reference" and this file
 *     is the pin, with seeded golden fixtures committed under tests/golden/.
 */
#ifndef VC_ORACLE_H
#define VC_ORACLE_H
#include <stdint.h>
#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Host threads the oracle's matvec/attention use (VCO_THREADS, else all cores). */
int vco_threads(void);

/* ---- scalar helpers (bit-exact with the device code) -------------------- */
uint64_t vco_splitmix64(uint64_t x);          /* util.hpp:30 restated */
float    vco_bf16_to_f32(uint16_t h);
uint16_t vco_f32_to_bf16(float f);            /* round to nearest even */
float    vco_f16_to_f32(uint16_t h);
uint16_t vco_f32_to_f16(float f);             /* round to nearest even */

/* Counter-based synthetic initialiser shared with the device init kernel:
 * value(i) = bf16( (float)(s_i - 131070) * k ), s_i = sum of the four 16-bit
 * lanes of splitmix64(seed ^ splitmix64(i + offset)), k = the float the
 * caller passes (std / (65536*sqrt(1/3)) rounded once to float). */
void vco_fill_normal_bf16(uint64_t seed, uint64_t offset, size_t n, float k, uint16_t* out);

/* ---- KIVI quantiser (per-channel K over token groups, per-token V over
 * channel groups; asymmetric min/max; fp16 scale and zero; RNE). -------- */
/* x: [rows][cols] bf16.  Quantises groups of `g` consecutive rows along the
 * row axis independently for every column (K: rows = tokens).  Writes one
 * code per byte: codes[rows][cols]; scale/zero: [rows/g][cols] fp16 bits.   */
void vco_quant_rows(const uint16_t* x, int rows, int cols, int g, int bits,
                    uint8_t* codes, uint16_t* scale, uint16_t* zero);
/* Quantises groups of `g` consecutive columns of every row (V: per token).
 * scale/zero: [rows][cols/g].                                              */
void vco_quant_cols(const uint16_t* x, int rows, int cols, int g, int bits,
                    uint8_t* codes, uint16_t* scale, uint16_t* zero);

/* ---- attention (fp64 accumulate) ----------------------------------------
 * One kv head, n_q query rows (fp32, already scaled by nothing), keys given
 * as fp32 arrays [n_keys][d].  Row r may see keys [0, lim[r]) (lim==NULL ->
 * all).  out: [n_q][d] fp32.  Softmax scale 1/sqrt(d).                     */
void vco_attention(const float* q, int n_q, const float* k, const float* v, int n_keys,
                   int d, const int* lim, float* out);

/* Dequantise a KIVI cache back to fp32 [T][d] (first nq_tokens rows from
 * codes, the rest copied from the bf16 tail).                              */
void vco_dequant_kv(const uint8_t* kcodes, const uint16_t* ks, const uint16_t* kz,
                    const uint8_t* vcodes, const uint16_t* vs, const uint16_t* vz,
                    int nq_tokens, int d, int gk, int gv,
                    const uint16_t* ktail, const uint16_t* vtail, int tail,
                    float* kout, float* vout);

/* ---- greedy argmax / accept / protocol ---------------------------------- */
int32_t vco_argmax(const float* logits, int n);   /* ties -> smallest index (specloop.cpp:260) */
/* specloop.cpp:37-56.  Returns number of accepted tokens written to out
 * (<= x+1); *first_mismatch = 1-based j or 0; *bonus = 1 when all matched. */
int vco_accept(const int32_t* drafted, const int32_t* preds, int x, int32_t* out,
               int* first_mismatch, int* bonus);

/* ---- top-k retention (drop-topk compressor) ----------------------------
 * Keep the k highest scores of scores[0..T) (ties -> lower position) and
 * write the kept positions ascending into kept[0..k).                      */
void vco_topk_kept(const float* scores, int T, int k, int32_t* kept);
/* Key-norm score used by the drop-topk compressor: s_t = sum_c |k_tc| * w_c
 * accumulated in channel order with IEEE fmaf (bit-exact with the device). */
void vco_key_scores(const uint16_t* k, int T, int d, const float* w, float* scores);

/* ---- drop-index generation (compressor.cpp:114-171 restated) ----------- */
/* std::mt19937_64 restated (the C++ standard fixes its output sequence).   */
typedef struct { uint64_t mt[312]; int idx; } vco_mt64;
void     vco_mt64_seed(vco_mt64* s, uint64_t seed);
uint64_t vco_mt64_next(vco_mt64* s);
/* Dropped positions for every (layer, head), layer-major, each sorted.
 * kind 0 = drop-uniform (seeded partial Fisher-Yates), 1 = drop-window.
 * out: [layers][heads][tokens - retained].  Returns drop count or -1.       */
int64_t vco_drop_indices(int kind, int layers, int heads, int64_t tokens, double ratio,
                         uint64_t seed, int sink_tokens, int64_t* out);

/* ---- tiny Llama-style model (config 1) --------------------------------- */
typedef struct {
  int vocab, hidden, layers, n_q, n_kv, d, ffn;
  float rope_theta, eps;
} vco_model_cfg;

/* Weights in logical layouts, bf16 bits:
 *   embed[vocab][hidden]; per layer: attn_norm[hidden],
 *   wqkv[(n_q+2n_kv)d][hidden] (q rows, then k rows, then v rows),
 *   wo[hidden][n_q d], mlp_norm[hidden], wgate[ffn][hidden], wup[ffn][hidden],
 *   wdown[hidden][ffn]; final_norm[hidden]; lm_head[vocab][hidden].       */
typedef struct {
  const uint16_t* embed;
  const uint16_t** attn_norm; const uint16_t** wqkv; const uint16_t** wo;
  const uint16_t** mlp_norm;  const uint16_t** wgate; const uint16_t** wup;
  const uint16_t** wdown;
  const uint16_t* final_norm; const uint16_t* lm_head;
} vco_model_weights;

/* Per-sequence KV as the oracle keeps it: fp32 views of what attention sees
 * for every layer/kv-head: k[layer][head][pos][d], v likewise, capacity cap.
 * `len` positions are valid.                                                */
typedef struct {
  float* k; float* v; int cap; int len;
} vco_kv;

/* Forward n tokens of one sequence at positions len..len+n-1 (causal among
 * themselves), appending their K/V (bf16-rounded, post-RoPE) to kv, writing
 * logits[n][vocab] and, when kv_out_k != NULL, the appended bf16 K/V bits
 * [layer][head][n][d].  rope_cos/sin: [max_pos][d/2] fp32 tables.          */
void vco_forward(const vco_model_cfg* cfg, const vco_model_weights* w, vco_kv* kv,
                 const int32_t* tokens, int n, const float* rope_cos, const float* rope_sin,
                 float* logits, uint16_t* kv_out_k, uint16_t* kv_out_v);

/* RoPE tables (double math, rounded once to float). */
void vco_rope_tables(int max_pos, int d, double theta, float* cos_out, float* sin_out);

#ifdef __cplusplus
}
#endif
#endif
