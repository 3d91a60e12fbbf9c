/*
 * ORACLE — TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, obviously-correct fp64 CPU definition of what ForkKV's
 * ResidualAttention computes. Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * It shares no code with the CUDA path (paper_2604_06370_b200/csrc).
 *
 * What it follows (PAPER.md = /root/reference/PAPER.md):
 *   Eq.1 (§2.2)       Y = xW + xA_iB_i
 *   Eq.2 (§2.2)       Y = bCache + rCache x B_i
 *   deferred RoPE (§2.2, §5.1, §5.3, Alg1.335):
 *        RoPE is applied to base K before caching; for the residual it is
 *        applied after the up-projection by B_k, at the key's absolute
 *        position.
 *   Alg.1 and Eq.4 compute, exactly up to rounding,
 *        softmax(Q K^T scale) (V_base + V_res B_v) with
 *        K = K_base + RoPE(K_res B_k).
 * The oracle is that plain definition written out: it MATERIALISES
 *        K[t] = Kb[t] + rho_t(Rk[t] . B_K^h)      (rho = identity in NONE mode)
 *        V[t] = Vb[t] + Rv[t] . B_V^h
 * per (sequence, kv head) and runs textbook softmax attention over the full
 * row (no blocking, no online softmax, no split).  Readings:
 *   C-2 RoPE pairing is NeoX half-split (i, i + d/2); inv_freq from the model
 *       rope config (plain theta^(-2i/d), or llama3 scaling).
 *   C-3 positions are absolute indices in the sequence, starting at 0.
 *   C-4 scale is passed in (1/sqrt(d) by default).
 *   C-5 one S and one (m, l): a single softmax over the full row.
 *   C-6 causal: query i of a chunk of C queries sits at p_i = L - C + i and
 *       sees keys t <= p_i; a row with no keys is an error (returns 6).
 *   C-7 LoRA alpha/r is folded into B by the caller.
 *
 * Build: gcc -O2 -shared -fPIC -o liboracle.so ra_oracle.c -lm -lpthread
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* --- RoPE frequencies (reading C-2) -------------------------------------
 * plain:  inv_freq[i] = theta^(-2i/d),  i = 0..d/2-1
 * llama3: the public Llama-3.1 rope_scaling rule (factor, low_freq_factor,
 *         high_freq_factor, original_max_position_embeddings): frequencies
 *         with wavelength < orig/high are kept, wavelength > orig/low are
 *         divided by factor, and the band in between is interpolated with
 *         smooth = (orig/wavelen - low) / (high - low).                    */
void oracle_inv_freq(int d, double theta, int llama3, double factor, double low,
                     double high, double orig, double* out) {
  for (int i = 0; i < d / 2; ++i) {
    double f = pow(theta, -2.0 * (double)i / (double)d);
    if (llama3) {
      double wavelen = 2.0 * M_PI / f;
      double low_wavelen = orig / low;
      double high_wavelen = orig / high;
      if (wavelen < high_wavelen) {
        /* keep */
      } else if (wavelen > low_wavelen) {
        f = f / factor;
      } else {
        double smooth = (orig / wavelen - low) / (high - low);
        f = (1.0 - smooth) * f / factor + smooth * f;
      }
    }
    out[i] = f;
  }
}

typedef struct {
  int L, C, Hq, Hkv, d, r, rope_mode;
  const double* inv_freq;
  const double *Kb, *Vb, *Rk, *Rv, *Bk, *Bv, *Q;
  double scale;
  double* O;
  double* lse;
  int h_begin, h_end;
  int status;
} job_t;

/* One kv head: materialise K, V for all L keys, then textbook attention for
 * every query head of the group and every query row. */
static void* run_heads(void* arg) {
  job_t* j = (job_t*)arg;
  const int L = j->L, C = j->C, d = j->d, r = j->r, Hkv = j->Hkv, Hq = j->Hq;
  const int g = Hq / Hkv;
  double* K = (double*)malloc(sizeof(double) * (size_t)L * d);
  double* V = (double*)malloc(sizeof(double) * (size_t)L * d);
  double* u = (double*)malloc(sizeof(double) * d);
  double* s = (double*)malloc(sizeof(double) * (size_t)(L > 0 ? L : 1));
  for (int h = j->h_begin; h < j->h_end; ++h) {
    const double* Bk = j->Bk + (size_t)h * r * d; /* B_K^h [r][d] */
    const double* Bv = j->Bv + (size_t)h * r * d; /* B_V^h [r][d] */
    for (int t = 0; t < L; ++t) {
      const double* rk = j->Rk + (size_t)t * r;
      const double* rv = j->Rv + (size_t)t * r;
      /* u = Rk[t] . B_K^h   (Eq.2 residual part, Alg1.335 K_res . B_k) */
      for (int e = 0; e < d; ++e) {
        double acc = 0.0;
        for (int q = 0; q < r; ++q) acc += rk[q] * Bk[(size_t)q * d + e];
        u[e] = acc;
      }
      /* rho_t: deferred RoPE at absolute position t (Alg1.335) */
      const double* kb = j->Kb + ((size_t)t * Hkv + h) * d;
      double* kr = K + (size_t)t * d;
      if (j->rope_mode == 1) {
        for (int i = 0; i < d / 2; ++i) {
          double ang = (double)t * j->inv_freq[i];
          double c = cos(ang), sn = sin(ang);
          double x0 = u[i], x1 = u[i + d / 2];
          kr[i] = kb[i] + (x0 * c - x1 * sn);
          kr[i + d / 2] = kb[i + d / 2] + (x0 * sn + x1 * c);
        }
      } else {
        for (int e = 0; e < d; ++e) kr[e] = kb[e] + u[e];
      }
      /* V[t] = Vb[t] + Rv[t] . B_V^h   (Eq.2 / Eq.4 left-hand side) */
      const double* vb = j->Vb + ((size_t)t * Hkv + h) * d;
      double* vr = V + (size_t)t * d;
      for (int e = 0; e < d; ++e) {
        double acc = 0.0;
        for (int q = 0; q < r; ++q) acc += rv[q] * Bv[(size_t)q * d + e];
        vr[e] = vb[e] + acc;
      }
    }
    for (int k = h * g; k < (h + 1) * g; ++k) {
      for (int i = 0; i < C; ++i) {
        const int p = L - C + i; /* C-6: absolute position of query i */
        const double* q = j->Q + ((size_t)i * Hq + k) * d;
        double* o = j->O + ((size_t)i * Hq + k) * d;
        if (p < 0) { j->status = 6; continue; }
        double m = -INFINITY;
        for (int t = 0; t <= p; ++t) {
          double acc = 0.0;
          for (int e = 0; e < d; ++e) acc += q[e] * K[(size_t)t * d + e];
          s[t] = acc * j->scale;
          if (s[t] > m) m = s[t];
        }
        double l = 0.0;
        for (int t = 0; t <= p; ++t) { s[t] = exp(s[t] - m); l += s[t]; }
        for (int e = 0; e < d; ++e) {
          double acc = 0.0;
          for (int t = 0; t <= p; ++t) acc += s[t] * V[(size_t)t * d + e];
          o[e] = acc / l;
        }
        if (j->lse) j->lse[(size_t)i * Hq + k] = m + log(l);
      }
    }
  }
  free(K); free(V); free(u); free(s);
  return NULL;
}

/*
 * oracle_residual_attention: one sequence.
 *   L       keys (sequence length, all keys 0..L-1)
 *   C       query rows: the last C positions of the sequence
 *   Kb, Vb  [L][Hkv][d]   base rows (Kb already RoPE'd at storage)
 *   Rk, Rv  [L][r]        residual rows (no RoPE)
 *   Bk, Bv  [Hkv][r][d]   per-kv-head column slices of B_K, B_V
 *   Q       [C][Hq][d]    RoPE'd queries
 *   O       [C][Hq][d]    output;  lse [C][Hq] optional (may be NULL)
 *   rope_mode 1 = DEFERRED (paper), 0 = NONE
 *   threads  number of pthreads over kv heads (<=0: 1)
 * returns 0, or 1 (bad shape), 6 (a query row with no keys).
 */
int oracle_residual_attention(int L, int C, int Hq, int Hkv, int d, int r, int rope_mode,
                              const double* inv_freq, const double* Kb, const double* Vb,
                              const double* Rk, const double* Rv, const double* Bk,
                              const double* Bv, const double* Q, double scale, double* O,
                              double* lse, int threads) {
  if (L < 0 || C < 0 || C > L || Hkv <= 0 || Hq % Hkv != 0 || d <= 0 || (d & 1) || r < 0)
    return 1;
  if (C == 0) return 0;
  if (L == 0) return 6;
  if (threads <= 0) threads = 1;
  if (threads > Hkv) threads = Hkv;
  pthread_t tid[256];
  job_t jobs[256];
  if (threads > 256) threads = 256;
  for (int w = 0; w < threads; ++w) {
    job_t* j = &jobs[w];
    j->L = L; j->C = C; j->Hq = Hq; j->Hkv = Hkv; j->d = d; j->r = r;
    j->rope_mode = rope_mode; j->inv_freq = inv_freq;
    j->Kb = Kb; j->Vb = Vb; j->Rk = Rk; j->Rv = Rv; j->Bk = Bk; j->Bv = Bv; j->Q = Q;
    j->scale = scale; j->O = O; j->lse = lse; j->status = 0;
    j->h_begin = (int)((long)Hkv * w / threads);
    j->h_end = (int)((long)Hkv * (w + 1) / threads);
    if (threads == 1) run_heads(j);
    else pthread_create(&tid[w], NULL, run_heads, j);
  }
  int st = 0;
  for (int w = 0; w < threads; ++w) {
    if (threads > 1) pthread_join(tid[w], NULL);
    if (jobs[w].status) st = jobs[w].status;
  }
  return st;
}
