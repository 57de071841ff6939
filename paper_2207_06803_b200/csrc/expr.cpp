// expr.cpp -- FFTc factorization expressions -> radix schedule (product path, host only).
//
// The paper's front end (Listing 1, Table 1) writes an FFT as a
// factorized matrix expression:
//     (DFT(2) ⊗ I(2)) · twiddle(4,2) · (I(2) ⊗ DFT(2)) · Permute(4,2) · InputComplex
// with ⊗ the Kronecker product, · the matrix product (right-associative), DFT(n),
// I(n), twiddle(N, M) = D^N_M and Permute(N, K) = Π^N_K (readings: DESIGN.md §2 #2).
// Here such an expression is parsed (recursive descent over our restatement of the
// grammar, Listing 2) and recognised as the paper's Eq. 2 applied recursively:
//     DFT_N = (DFT_K ⊗ I_M) · D^N_M · (I_K ⊗ X_M) · Π^N_K,   N = M K,
// where X_M is DFT(M) or again such a factorization.  The result is the radix schedule
// R_0 ... R_{S-1} (R_0 = the innermost DFT, the last = the outermost K) that the GPU
// executes as Stockham stages, each stage one level of Eq. 2 (fused.cuh).  A factored
// outer DFT_K is flattened into consecutive stages (its radices, innermost first).
// A bare DFT(N) leaves the choice of radices to the planner.
//
// Accepted spellings: '·' (U+00B7), '*' or '@' for the product; '⊗' (U+2297) or '&' for
// the Kronecker product; DFT/dft/F, I/Id/identity, twiddle/D/T, Permute/permute/P/L.
// An optional "var name =" prefix, a trailing ';' and a trailing input identifier
// (Listing 1's "· InputComplex") are accepted and ignored.
#include <ctype.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include <memory>
#include <string>
#include <vector>

#include "expr.h"
#include "planner.h"

namespace fftc {

namespace {

enum NodeKind { N_DFT, N_ID, N_TW, N_PERM, N_KRON, N_MUL, N_INPUT };

struct Node {
  NodeKind k;
  int64_t a = 0, b = 0;                     // DFT(a), I(a), twiddle(a, b), Permute(a, b)
  std::vector<std::unique_ptr<Node>> kids;  // KRON: 2, MUL: >= 2 (left to right)
};

struct Parser {
  const char* s;
  size_t i = 0;
  std::string err;
  int depth = 0;  // parenthesis nesting (bounded: the recursion stays on a small stack)

  void ws() {
    while (s[i] && isspace((unsigned char)s[i])) ++i;
  }
  bool fail(const std::string& m) {
    if (err.empty()) {
      char buf[64];
      snprintf(buf, sizeof buf, " (at offset %zu)", i);
      err = m + buf;
    }
    return false;
  }
  // matrix product operator: '·' (C2 B7), '*', '@'
  bool mul_op() {
    ws();
    if (s[i] == '*' || s[i] == '@') {
      ++i;
      return true;
    }
    if ((unsigned char)s[i] == 0xC2 && (unsigned char)s[i + 1] == 0xB7) {
      i += 2;
      return true;
    }
    return false;
  }
  // Kronecker operator: '⊗' (E2 8A 97) or '&'
  bool kron_op() {
    ws();
    if (s[i] == '&') {
      ++i;
      return true;
    }
    if ((unsigned char)s[i] == 0xE2 && (unsigned char)s[i + 1] == 0x8A && (unsigned char)s[i + 2] == 0x97) {
      i += 3;
      return true;
    }
    return false;
  }
  bool integer(int64_t* v) {
    ws();
    if (!isdigit((unsigned char)s[i])) return fail("expected an integer");
    int64_t x = 0;
    while (isdigit((unsigned char)s[i])) {
      x = x * 10 + (s[i] - '0');
      if (x > ((int64_t)1 << 40)) return fail("integer too large");
      ++i;
    }
    *v = x;
    return true;
  }
  bool ident(std::string* id) {
    ws();
    if (!isalpha((unsigned char)s[i]) && s[i] != '_') return false;
    size_t j = i;
    while (isalnum((unsigned char)s[j]) || s[j] == '_') ++j;
    id->assign(s + i, j - i);
    i = j;
    return true;
  }
  bool expect(char c) {
    ws();
    if (s[i] != c) {
      char m[32];
      snprintf(m, sizeof m, "expected '%c'", c);
      return fail(m);
    }
    ++i;
    return true;
  }
  // factor := NAME '(' int [',' int] ')' | '(' expr ')' | input-identifier
  std::unique_ptr<Node> factor() {
    ws();
    if (s[i] == '(') {
      if (++depth > 64) {
        fail("nesting deeper than 64");
        return nullptr;
      }
      ++i;
      auto e = expr();
      --depth;
      if (!e || !expect(')')) return nullptr;
      return e;
    }
    std::string id;
    if (!ident(&id)) {
      fail("expected DFT, I, twiddle, Permute or '('");
      return nullptr;
    }
    ws();
    auto n = std::make_unique<Node>();
    if (s[i] != '(') {  // a bare identifier: the input vector of Listing 1
      n->k = N_INPUT;
      return n;
    }
    int nargs = 0;
    if (id == "DFT" || id == "dft" || id == "F") n->k = N_DFT, nargs = 1;
    else if (id == "I" || id == "Id" || id == "identity") n->k = N_ID, nargs = 1;
    else if (id == "twiddle" || id == "D" || id == "T") n->k = N_TW, nargs = 2;
    else if (id == "Permute" || id == "permute" || id == "P" || id == "L") n->k = N_PERM, nargs = 2;
    else {
      fail("unknown operator '" + id + "'");
      return nullptr;
    }
    ++i;  // '('
    if (!integer(&n->a)) return nullptr;
    if (nargs == 2 && (!expect(',') || !integer(&n->b))) return nullptr;
    if (!expect(')')) return nullptr;
    return n;
  }
  // term := factor ('⊗' factor)*   (left-associative)
  std::unique_ptr<Node> term() {
    auto l = factor();
    if (!l) return nullptr;
    int nk = 0;
    while (kron_op()) {
      if (++nk > 64) {
        fail("more than 64 Kronecker factors");
        return nullptr;
      }
      auto r = factor();
      if (!r) return nullptr;
      auto k = std::make_unique<Node>();
      k->k = N_KRON;
      k->kids.push_back(std::move(l));
      k->kids.push_back(std::move(r));
      l = std::move(k);
    }
    return l;
  }
  // expr := term ('·' term)*   (a product chain; associativity is immaterial for its value)
  std::unique_ptr<Node> expr() {
    auto l = term();
    if (!l) return nullptr;
    if (!mul_op()) return l;
    auto m = std::make_unique<Node>();
    m->k = N_MUL;
    m->kids.push_back(std::move(l));
    do {
      if (m->kids.size() > 256) {
        fail("more than 256 product factors");
        return nullptr;
      }
      auto r = term();
      if (!r) return nullptr;
      m->kids.push_back(std::move(r));
    } while (mul_op());
    // a parenthesised product inside a product chain is the same chain (associativity)
    std::vector<std::unique_ptr<Node>> flat;
    for (auto& k : m->kids) {
      if (k->k == N_MUL)
        for (auto& kk : k->kids) flat.push_back(std::move(kk));
      else
        flat.push_back(std::move(k));
    }
    m->kids = std::move(flat);
    return m;
  }
};

// Size (rows) of a matrix node, or -1.
int64_t dim(const Node* n) {
  switch (n->k) {
    case N_DFT:
    case N_ID:
    case N_TW:
    case N_PERM: return n->a;
    case N_KRON: {
      const int64_t a = dim(n->kids[0].get()), b = dim(n->kids[1].get());
      return (a < 0 || b < 0) ? -1 : a * b;
    }
    case N_MUL: return dim(n->kids[0].get());
    default: return -1;
  }
}

// Match n as a factorization of DFT_N; append its radices (innermost first) to out.
// A DFT(n) leaf appends n (or, at the top level only, is left to the planner).
bool lower(const Node* n, int64_t* N, std::vector<int64_t>* out, std::string* err) {
  if (n->k == N_DFT) {
    if (n->a < 1) {
      *err = "DFT(n) needs n >= 1";
      return false;
    }
    *N = n->a;
    if (n->a > 1) out->push_back(n->a);
    return true;
  }
  if (n->k != N_MUL || n->kids.size() != 4) {
    *err = "not a Cooley-Tukey factorization: expected (DFT_K ⊗ I_M) · twiddle(N, M) · (I_K ⊗ X_M) · Permute(N, K)";
    return false;
  }
  const Node* A = n->kids[0].get();
  const Node* Dn = n->kids[1].get();
  const Node* C = n->kids[2].get();
  const Node* P = n->kids[3].get();
  if (A->k != N_KRON || A->kids[1]->k != N_ID) {
    *err = "first factor must be (DFT_K ⊗ I_M)";
    return false;
  }
  if (C->k != N_KRON || C->kids[0]->k != N_ID) {
    *err = "third factor must be (I_K ⊗ X_M)";
    return false;
  }
  if (Dn->k != N_TW) {
    *err = "second factor must be twiddle(N, M)";
    return false;
  }
  if (P->k != N_PERM) {
    *err = "fourth factor must be Permute(N, K)";
    return false;
  }
  const int64_t M = A->kids[1]->a, K = C->kids[0]->a;
  int64_t Kin = 0, Min = 0;
  std::vector<int64_t> rk, rm;
  if (!lower(A->kids[0].get(), &Kin, &rk, err)) return false;       // DFT_K (or a factorization)
  if (!lower(C->kids[1].get(), &Min, &rm, err)) return false;       // X_M
  const int64_t NN = K * M;
  char buf[160];
  if (Kin != K || Min != M || Dn->a != NN || Dn->b != M || P->a != NN || P->b != K) {
    snprintf(buf, sizeof buf,
             "sizes do not form Eq. 2: DFT_%lld ⊗ I_%lld, twiddle(%lld,%lld), I_%lld ⊗ DFT_%lld, Permute(%lld,%lld)",
             (long long)Kin, (long long)M, (long long)Dn->a, (long long)Dn->b, (long long)K, (long long)Min,
             (long long)P->a, (long long)P->b);
    *err = buf;
    return false;
  }
  *N = NN;
  out->insert(out->end(), rm.begin(), rm.end());  // the inner DFT_M first ...
  out->insert(out->end(), rk.begin(), rk.end());  // ... then the outer DFT_K
  return true;
}

}  // namespace

int expr_radices(const char* text, int64_t* N, int64_t* radices, int max, char* err, size_t errlen) {
  auto set_err = [&](const std::string& m) {
    if (err && errlen) {
      strncpy(err, m.c_str(), errlen - 1);
      err[errlen - 1] = 0;
    }
    return -1;
  };
  if (!text || !N) return set_err("NULL argument");
  std::string src(text);
  // optional "var name =" prefix and trailing ';'
  size_t p = src.find_first_not_of(" \t\r\n");
  if (p != std::string::npos && src.compare(p, 4, "var ") == 0) {
    const size_t eq = src.find('=', p);
    if (eq == std::string::npos) return set_err("'var' without '='");
    src = src.substr(eq + 1);
  }
  while (!src.empty() && (isspace((unsigned char)src.back()) || src.back() == ';')) src.pop_back();
  Parser ps{src.c_str()};
  auto root = ps.expr();
  if (!root) return set_err(ps.err);
  ps.ws();
  if (ps.s[ps.i]) {
    ps.fail("unexpected trailing text");
    return set_err(ps.err);
  }
  // drop a trailing input identifier (Listing 1: "... · Permute(4,2) · InputComplex")
  if (root->k == N_MUL && root->kids.back()->k == N_INPUT) {
    root->kids.pop_back();
    if (root->kids.size() == 1) {
      std::unique_ptr<Node> only = std::move(root->kids[0]);
      root = std::move(only);
    }
  }
  if (root->k == N_INPUT) return set_err("expression has no matrix factors");
  std::vector<int64_t> r;
  std::string e;
  int64_t n = 0;
  if (root->k == N_DFT) {  // a bare DFT(N): the planner chooses
    if (root->a < 1) return set_err("DFT(n) needs n >= 1");
    *N = root->a;
    return 0;
  }
  if (!lower(root.get(), &n, &r, &e)) return set_err(e);
  if (dim(root.get()) != n) return set_err("inconsistent matrix sizes");
  *N = n;
  if ((int)r.size() > max) return set_err("too many stages");
  for (size_t k = 0; k < r.size(); ++k) radices[k] = r[k];
  return (int)r.size();
}

}  // namespace fftc
