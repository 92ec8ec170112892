// gn_io.cpp -- native parser of the DIMACS-flavoured MWIS instance text
// (reference io.py:43-102 parse_instance).
//
//   c optional comments
//   p mwis <n> <m>
//   n <vertex-id> <weight>     (ids 1-based)
//   e <u> <v>                  (ids 1-based)
//
// The text is walked line by line exactly as parse_instance walks
// text.splitlines(): the same checks in the same order, the first failing
// line wins, and the error text is the reference's FormatError message
// (line numbers, Python repr of the stripped line or token).  Then the
// post-checks of io.py:87-96 (problem line present, edge count, first vertex
// without a weight).  Weights are parsed with strtod (correctly rounded, as
// Python's float()); ids and counts as 64-bit integers.
//
// The native grammar is the format's ASCII one.  Text the Python built-ins
// would read differently from a C scanner -- non-ASCII or control bytes
// other than \t \n \r (str.strip/split/splitlines know more whitespace and
// line breaks), '_' (PEP 515 digit separators in int()/float()), integers of
// more than 18 digits, a vertex count above 2^31, and error lines whose repr
// needs quoting rules (quotes, backslashes) -- returns GN_PARSE_FALLBACK
// before any work is wasted on it; io.py then runs its reference-identical
// Python parser on that text.
#include <cerrno>
#include <cmath>
#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "gn_b200.h"

struct gn_mwis {
    int64_t n = 0, m = 0;
    std::vector<double> w;       // [n], 1-based id i at w[i-1]
    std::vector<int64_t> eu, ev;  // 0-based endpoints, file order
};

namespace {

struct Tok {
    const char* p;
    int64_t len;
    bool eq(const char* s) const { return (int64_t)strlen(s) == len && memcmp(p, s, (size_t)len) == 0; }
    std::string str() const { return std::string(p, (size_t)len); }
};

// Python repr() of an ASCII string without quotes or backslashes: '...' with
// tabs escaped.  Returns false when repr would need other quoting.
bool py_repr(const char* p, int64_t len, std::string& out) {
    out = "'";
    for (int64_t i = 0; i < len; ++i) {
        const char c = p[i];
        if (c == '\'' || c == '"' || c == '\\') return false;
        if (c == '\t') out += "\\t";
        else out += c;
    }
    out += "'";
    return true;
}

enum { kNum = 0, kBad = 1, kFallback = 2 };

// int(): [+-]?[0-9]+ (at most 18 digits here)
int parse_int(const Tok& t, int64_t* v) {
    int64_t i = 0;
    bool neg = false;
    if (i < t.len && (t.p[i] == '+' || t.p[i] == '-')) neg = t.p[i++] == '-';
    if (i == t.len) return kBad;
    if (t.len - i > 18) {
        for (int64_t k = i; k < t.len; ++k)
            if (t.p[k] < '0' || t.p[k] > '9') return kBad;
        return kFallback;  // Python ints are unbounded
    }
    int64_t x = 0;
    for (; i < t.len; ++i) {
        if (t.p[i] < '0' || t.p[i] > '9') return kBad;
        x = x * 10 + (t.p[i] - '0');
    }
    *v = neg ? -x : x;
    return kNum;
}

bool ieq(const char* p, int64_t len, const char* s) {
    if ((int64_t)strlen(s) != len) return false;
    for (int64_t i = 0; i < len; ++i) {
        char c = p[i];
        if (c >= 'A' && c <= 'Z') c = (char)(c - 'A' + 'a');
        if (c != s[i]) return false;
    }
    return true;
}

// float(): [+-]? (digits [. digits?] | . digits) ([eE] [+-]? digits)?, or
// inf / infinity / nan in any case
int parse_float(const Tok& t, double* v) {
    int64_t i = 0;
    bool neg = false;
    if (i < t.len && (t.p[i] == '+' || t.p[i] == '-')) neg = t.p[i++] == '-';
    const char* b = t.p + i;
    const int64_t bl = t.len - i;
    if (ieq(b, bl, "inf") || ieq(b, bl, "infinity")) {
        *v = neg ? -INFINITY : INFINITY;
        return kNum;
    }
    if (ieq(b, bl, "nan")) {
        *v = neg ? -NAN : NAN;
        return kNum;
    }
    int64_t k = i, d1 = 0, d2 = 0;
    while (k < t.len && t.p[k] >= '0' && t.p[k] <= '9') ++k, ++d1;
    if (k < t.len && t.p[k] == '.') {
        ++k;
        while (k < t.len && t.p[k] >= '0' && t.p[k] <= '9') ++k, ++d2;
    }
    if (d1 + d2 == 0) return kBad;
    if (k < t.len && (t.p[k] == 'e' || t.p[k] == 'E')) {
        ++k;
        if (k < t.len && (t.p[k] == '+' || t.p[k] == '-')) ++k;
        int64_t d3 = 0;
        while (k < t.len && t.p[k] >= '0' && t.p[k] <= '9') ++k, ++d3;
        if (d3 == 0) return kBad;
    }
    if (k != t.len) return kBad;
    const std::string s = t.str();
    errno = 0;
    *v = strtod(s.c_str(), nullptr);  // correctly rounded; overflow gives +-inf like float()
    return kNum;
}

}  // namespace

extern "C" {

int gn_mwis_parse(const char* text, int64_t len, gn_mwis** out, char* err, int64_t err_len) {
    if (!out || (len > 0 && !text)) return GN_ERR_ARG;
    *out = nullptr;
    auto set_err = [&](const std::string& msg) {
        if (err && err_len > 0) snprintf(err, (size_t)err_len, "%s", msg.c_str());
        return GN_ERR_FORMAT;
    };
    // characters whose meaning the Python built-ins extend: the Python parser takes those texts
    for (int64_t i = 0; i < len; ++i) {
        const unsigned char c = (unsigned char)text[i];
        if ((c < 0x20 && c != '\t' && c != '\n' && c != '\r') || c >= 0x7f || c == '_') return GN_PARSE_FALLBACK;
    }
    gn_mwis* R = new gn_mwis();
    std::vector<uint8_t> have;
    bool has_p = false;
    int64_t pos = 0, lineno = 0;
    std::string rep;
    auto fallback = [&]() {
        delete R;
        return GN_PARSE_FALLBACK;
    };
    auto error = [&](const std::string& msg) {
        delete R;
        return set_err(msg);
    };
    Tok tk[5];
    while (pos < len) {
        int64_t e = pos;
        while (e < len && text[e] != '\n' && text[e] != '\r') ++e;
        const int64_t next = (e < len && text[e] == '\r' && e + 1 < len && text[e + 1] == '\n') ? e + 2 : e + 1;
        ++lineno;
        int64_t a = pos, z = e;  // strip()
        while (a < z && (text[a] == ' ' || text[a] == '\t')) ++a;
        while (z > a && (text[z - 1] == ' ' || text[z - 1] == '\t')) --z;
        pos = next;
        if (a == z || text[a] == 'c') continue;
        int nt = 0;  // split(), at most 5 tokens kept (more only matters as "wrong count")
        for (int64_t q = a; q < z;) {
            while (q < z && (text[q] == ' ' || text[q] == '\t')) ++q;
            if (q >= z) break;
            int64_t r = q;
            while (r < z && text[r] != ' ' && text[r] != '\t') ++r;
            if (nt < 5) tk[nt] = Tok{text + q, r - q};
            ++nt;
            q = r;
        }
        const std::string ln = "line " + std::to_string(lineno) + ": ";
        auto line_repr = [&]() { return py_repr(text + a, z - a, rep); };
        const Tok& kind = tk[0];
        if (kind.eq("p")) {
            if (nt != 4 || !tk[1].eq("mwis")) {
                if (!line_repr()) return fallback();
                return error(ln + "malformed problem line " + rep);
            }
            if (has_p) return error(ln + "duplicate problem line");
            int64_t n = 0, m = 0;
            int r1 = parse_int(tk[2], &n);
            if (r1 == kNum) r1 = parse_int(tk[3], &m);
            if (r1 == kFallback) return fallback();
            if (r1 == kBad) {
                if (!line_repr()) return fallback();
                return error(ln + "cannot parse number in " + rep);
            }
            if (n > (int64_t(1) << 31)) return fallback();
            has_p = true;
            R->n = n;
            R->m = m;
            R->w.assign((size_t)std::max<int64_t>(n, 0), 0.0);
            have.assign((size_t)std::max<int64_t>(n, 0), 0);
        } else if (kind.eq("n")) {
            if (!has_p) return error(ln + "weight line before problem line");
            if (nt != 3) {
                if (!line_repr()) return fallback();
                return error(ln + "malformed weight line " + rep);
            }
            int64_t vid = 0;
            int r1 = parse_int(tk[1], &vid);
            if (r1 == kFallback) return fallback();
            if (r1 == kBad) {
                if (!line_repr()) return fallback();
                return error(ln + "cannot parse number in " + rep);
            }
            if (!(1 <= vid && vid <= R->n))
                return error(ln + "vertex id " + std::to_string(vid) + " outside 1.." + std::to_string(R->n));
            if (have[(size_t)(vid - 1)]) return error(ln + "duplicate weight for vertex " + std::to_string(vid));
            double wv = 0.0;
            const int r2 = parse_float(tk[2], &wv);
            if (r2 != kNum) {
                if (!line_repr()) return fallback();
                return error(ln + "cannot parse number in " + rep);
            }
            have[(size_t)(vid - 1)] = 1;
            R->w[(size_t)(vid - 1)] = wv;
        } else if (kind.eq("e")) {
            if (!has_p) return error(ln + "edge line before problem line");
            if (nt != 3) {
                if (!line_repr()) return fallback();
                return error(ln + "malformed edge line " + rep);
            }
            int64_t u = 0, v = 0;
            int r1 = parse_int(tk[1], &u);
            if (r1 == kNum) r1 = parse_int(tk[2], &v);
            if (r1 == kFallback) return fallback();
            if (r1 == kBad) {
                if (!line_repr()) return fallback();
                return error(ln + "cannot parse number in " + rep);
            }
            if (!(1 <= u && u <= R->n && 1 <= v && v <= R->n))
                return error(ln + "edge (" + std::to_string(u) + "," + std::to_string(v) + ") outside 1.." +
                             std::to_string(R->n));
            R->eu.push_back(u - 1);
            R->ev.push_back(v - 1);
        } else {
            if (!py_repr(kind.p, kind.len, rep)) return fallback();
            return error(ln + "unknown line type " + rep);
        }
    }
    // io.py:87-96
    if (!has_p) return error("missing problem line");
    if ((int64_t)R->eu.size() != R->m)
        return error("problem line declares " + std::to_string(R->m) + " edges, file has " +
                     std::to_string(R->eu.size()));
    for (int64_t i = 0; i < R->n; ++i)
        if (!have[(size_t)i]) return error("missing weight for vertex " + std::to_string(i + 1));
    *out = R;
    return GN_OK;
}

int gn_mwis_info(const gn_mwis* r, int64_t* n, int64_t* m) {
    if (!r) return GN_ERR_ARG;
    if (n) *n = r->n;
    if (m) *m = (int64_t)r->eu.size();
    return GN_OK;
}

int gn_mwis_copy(const gn_mwis* r, double* w, int64_t* edges) {
    if (!r) return GN_ERR_ARG;
    if (w && r->n > 0) memcpy(w, r->w.data(), sizeof(double) * (size_t)r->n);
    if (edges)
        for (size_t k = 0; k < r->eu.size(); ++k) {
            edges[2 * k] = r->eu[k];
            edges[2 * k + 1] = r->ev[k];
        }
    return GN_OK;
}

void gn_mwis_free(gn_mwis* r) { delete r; }

}  // extern "C"
