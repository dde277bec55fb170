// textio.cpp -- host-side ingest of the reference's plain-text formats straight
// into packed adjacency rows (the layout Graph._packed holds, graph.py:78-88).
//
// Replaces, byte for byte in behaviour:
//   parse_graph_text     textio.py:30-86  (strict: comments "c...", header
//                        "p <n> <m>", exactly m lines "e <u> <v>"; the first
//                        offending line is reported with the reference's
//                        message and 1-based line number)
//   write_graph_text     textio.py:89-93  (edges u < v ascending)
//   parse_ordering_text  textio.py:96-106
//   write_ordering_text  textio.py:109-110
// The reference decodes UTF-8 and then uses str.splitlines / str.strip /
// str.split / int(); the scanner below applies the same rules to the UTF-8
// bytes: line breaks \n \r \r\n \v \f \x1c \x1d \x1e U+0085 U+2028 U+2029,
// whitespace = those plus \t, space, \x1f and the Unicode space separators,
// integers = optional sign, ASCII digits with single underscores between
// digits (int() also accepts non-ASCII decimal digits; such fields are
// rejected here as non-integers -- the only documented difference).
// Duplicate edges are detected on the rows being filled (a bit already set),
// so parsing and building the Graph are one pass; the reference builds its
// rows afterwards with np.unique + bitwise_or.at (graph.py:80-88).
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/chordal_b200.h"

namespace {

// ---- UTF-8 classification ----------------------------------------------------

// Length of a valid UTF-8 sequence at p (1-4) or 0 if invalid.
int utf8_len(const unsigned char *p, const unsigned char *end) {
    const unsigned c = p[0];
    if (c < 0x80) return 1;
    auto cont = [&](int k) { return p + k < end && (p[k] & 0xC0) == 0x80; };
    if (c >= 0xC2 && c <= 0xDF) return cont(1) ? 2 : 0;
    if (c >= 0xE0 && c <= 0xEF) {
        if (!cont(1) || !cont(2)) return 0;
        if (c == 0xE0 && p[1] < 0xA0) return 0;   // overlong
        if (c == 0xED && p[1] >= 0xA0) return 0;  // surrogates
        return 3;
    }
    if (c >= 0xF0 && c <= 0xF4) {
        if (!cont(1) || !cont(2) || !cont(3)) return 0;
        if (c == 0xF0 && p[1] < 0x90) return 0;
        if (c == 0xF4 && p[1] >= 0x90) return 0;
        return 4;
    }
    return 0;
}

// Line break at p (str.splitlines): length in bytes, 0 if none.  \r\n is one.
int line_break(const unsigned char *p, const unsigned char *end) {
    const unsigned c = p[0];
    if (c == '\n' || c == '\v' || c == '\f' || c == 0x1C || c == 0x1D || c == 0x1E) return 1;
    if (c == '\r') return (p + 1 < end && p[1] == '\n') ? 2 : 1;
    if (c == 0xC2 && p + 1 < end && p[1] == 0x85) return 2;  // U+0085
    if (c == 0xE2 && p + 2 < end && p[1] == 0x80 && (p[2] == 0xA8 || p[2] == 0xA9)) return 3;  // U+2028/9
    return 0;
}

// In-line whitespace at p (str.split / str.strip, after line splitting): length or 0.
int space_at(const unsigned char *p, const unsigned char *end) {
    const unsigned c = p[0];
    if (c == ' ' || c == '\t' || c == 0x1F) return 1;
    if (c < 0x80) return 0;
    if (c == 0xC2 && p + 1 < end && p[1] == 0xA0) return 2;                              // U+00A0
    if (c == 0xE1 && p + 2 < end && p[1] == 0x9A && p[2] == 0x80) return 3;              // U+1680
    if (c == 0xE2 && p + 2 < end && p[1] == 0x80 && (p[2] <= 0x8A || p[2] == 0xAF)) return 3;  // U+2000-200A, 202F
    if (c == 0xE2 && p + 2 < end && p[1] == 0x81 && p[2] == 0x9F) return 3;              // U+205F
    if (c == 0xE3 && p + 2 < end && p[1] == 0x80 && p[2] == 0x80) return 3;              // U+3000
    return 0;
}

struct Field {
    const unsigned char *b, *e;
    bool is(const char *s) const { return (size_t)(e - b) == strlen(s) && memcmp(b, s, e - b) == 0; }
};

// Splits [b, e) at whitespace into at most `cap` fields; returns the field count
// (counting beyond cap so "wrong number of fields" is detected).
int split_fields(const unsigned char *b, const unsigned char *e, Field *out, int cap) {
    int k = 0;
    const unsigned char *p = b;
    while (p < e) {
        int s;
        while (p < e && (s = space_at(p, e)) > 0) p += s;
        if (p >= e) break;
        const unsigned char *fb = p;
        while (p < e && space_at(p, e) == 0) p += (*p < 0x80) ? 1 : (utf8_len(p, e) ? utf8_len(p, e) : 1);
        if (k < cap) out[k] = Field{fb, p};
        ++k;
    }
    return k;
}

// Python int() on an already-split field: [+-] digit (['_'] digit)*.
// Produces the canonical decimal text (as Python prints the value) and the value
// saturated to int64 range (`big` set when it does not fit).
bool parse_int(const Field &f, std::string &canon, long long &val, bool &big) {
    const unsigned char *p = f.b, *e = f.e;
    bool neg = false;
    if (p < e && (*p == '+' || *p == '-')) {
        neg = *p == '-';
        ++p;
    }
    if (p >= e || *p < '0' || *p > '9') return false;
    std::string digits;
    bool prev_us = false;
    for (; p < e; ++p) {
        if (*p >= '0' && *p <= '9') {
            digits.push_back((char)*p);
            prev_us = false;
        } else if (*p == '_' && !prev_us && !digits.empty()) {
            prev_us = true;
        } else {
            return false;
        }
    }
    if (prev_us) return false;
    size_t z = 0;
    while (z + 1 < digits.size() && digits[z] == '0') ++z;
    digits.erase(0, z);
    const bool zero = digits == "0";
    canon = (neg && !zero ? "-" : "") + digits;
    big = false;
    unsigned long long acc = 0;
    for (char c : digits) {
        if (acc > (0x7FFFFFFFFFFFFFFFULL - (unsigned)(c - '0')) / 10) {
            big = true;
            break;
        }
        acc = acc * 10 + (unsigned)(c - '0');
    }
    if (big) acc = 0x7FFFFFFFFFFFFFFFULL;
    val = neg ? -(long long)acc : (long long)acc;
    return true;
}

struct Err {
    int status = CHORDAL_OK;
    long long line = -1;
    std::string msg;
};

void put_err(const Err &er, int64_t *err_line, char *err_msg, int64_t err_cap) {
    if (err_line) *err_line = er.line;
    if (err_msg && err_cap > 0) {
        const size_t k = std::min<size_t>(er.msg.size(), (size_t)err_cap - 1);
        memcpy(err_msg, er.msg.data(), k);
        err_msg[k] = 0;
    }
}

}  // namespace

extern "C" {

int chordal_parse_graph_text(const char *text, int64_t len, int64_t cap, int64_t *n_out, int64_t *m_out,
                             uint8_t *rows_out, int64_t row_bytes, int64_t *err_line, char *err_msg,
                             int64_t err_cap) {
    if (len < 0 || (len > 0 && !text) || !n_out || !m_out) return CHORDAL_EINVAL;
    const unsigned char *p = reinterpret_cast<const unsigned char *>(text), *end = p + len;
    Err er;
    auto fail = [&](int status, long long line, std::string msg) {
        er.status = status;
        er.line = line;
        er.msg = std::move(msg);
        put_err(er, err_line, err_msg, err_cap);
        return status;
    };
    // the reference decodes first: any invalid UTF-8 anywhere fails before parsing
    for (const unsigned char *q = p; q < end;) {
        if (*q < 0x80) { ++q; continue; }
        const int k = utf8_len(q, end);
        if (!k) return fail(CHORDAL_EUTF8, -1, "input is not valid UTF-8");
        q += k;
    }
    long long n = -1, m = -1, header_line = 0, edges_seen = 0, lineno = 0;
    std::string n_canon, m_canon;
    const bool fill = rows_out != nullptr;
    if (fill && row_bytes < 0) return CHORDAL_EINVAL;
    Field f[4];
    while (p < end) {
        // Fast path for the common edge line: [spaces] 'e' spaces digits spaces
        // digits [spaces] (break | end), all ASCII, values < 10^9.  Anything else
        // (and every check that fails) goes through the general path below.
        if (fill && n >= 0) {
            const unsigned char *q = p;
            while (q < end && (*q == ' ' || *q == '\t')) ++q;
            if (q + 1 < end && q[0] == 'e' && (q[1] == ' ' || q[1] == '\t')) {
                ++q;
                long long a = 0, b = 0;
                int da = 0, db = 0;
                while (q < end && (*q == ' ' || *q == '\t')) ++q;
                while (q < end && *q >= '0' && *q <= '9' && da < 10) { a = 10 * a + (*q - '0'); ++q; ++da; }
                const unsigned char *qa = q;
                while (q < end && (*q == ' ' || *q == '\t')) ++q;
                const bool sep = q > qa;
                while (q < end && *q >= '0' && *q <= '9' && db < 10) { b = 10 * b + (*q - '0'); ++q; ++db; }
                while (q < end && (*q == ' ' || *q == '\t')) ++q;
                int brk = 0;
                const bool at_end = q >= end || (*q < 0x80 && (brk = line_break(q, end)) > 0);
                if (da && db && da < 10 && db < 10 && sep && at_end && a >= 1 && a <= n && b >= 1 && b <= n &&
                    a != b) {
                    const long long lo = a < b ? a : b, hi = a < b ? b : a;
                    uint8_t *rl = rows_out + (lo - 1) * row_bytes;
                    const long long hb = hi - 1, lbit = lo - 1;
                    if (!((rl[hb >> 3] >> (hb & 7)) & 1) && edges_seen < m) {
                        ++edges_seen;
                        ++lineno;
                        rl[hb >> 3] |= (uint8_t)(1u << (hb & 7));
                        rows_out[hb * row_bytes + (lbit >> 3)] |= (uint8_t)(1u << (lbit & 7));
                        p = q + brk;
                        continue;
                    }
                }
            }
        }
        // one line [p, le), then its break
        const unsigned char *lb = p;
        int brk = 0;
        while (p < end && (brk = line_break(p, end)) == 0) p += (*p < 0x80) ? 1 : utf8_len(p, end);
        const unsigned char *le = p;
        p += brk;
        ++lineno;
        // strip
        int s;
        while (lb < le && (s = space_at(lb, le)) > 0) lb += s;
        if (lb == le || *lb == 'c') continue;
        const int nf = split_fields(lb, le, f, 4);
        if (n < 0) {
            if (!f[0].is("p") || nf != 3) return fail(CHORDAL_EPARSE, lineno, "expected header 'p <n> <m>'");
            long long nv, mv;
            bool nb, mb;
            if (!parse_int(f[1], n_canon, nv, nb) || !parse_int(f[2], m_canon, mv, mb))
                return fail(CHORDAL_EPARSE, lineno, "header counts must be integers");
            if (nv < 0 || mv < 0) return fail(CHORDAL_EPARSE, lineno, "header counts must be non-negative");
            // _check_size(n, cap) (graph.py:23-28): the caller formats GraphTooLarge
            if (nb || (cap >= 0 && nv > cap)) {
                *n_out = nb ? -1 : nv;
                return fail(CHORDAL_ETOOLARGE, lineno, n_canon);
            }
            n = nv;
            m = mb ? 0x7FFFFFFFFFFFFFFFLL : mv;
            header_line = lineno;
            *n_out = n;
            *m_out = m;
            if (!fill) return CHORDAL_OK;  // header-only call: the caller sizes the rows
            continue;
        }
        if (!f[0].is("e") || nf != 3) return fail(CHORDAL_EPARSE, lineno, "expected edge line 'e <u> <v>'");
        std::string uc, vc;
        long long u, v;
        bool ub, vb;
        if (!parse_int(f[1], uc, u, ub) || !parse_int(f[2], vc, v, vb))
            return fail(CHORDAL_EPARSE, lineno, "edge endpoints must be integers");
        if (ub || vb || !(1 <= u && u <= n && 1 <= v && v <= n))
            return fail(CHORDAL_EPARSE, lineno,
                        "edge (" + uc + ", " + vc + ") outside vertex range 1.." + std::to_string(n));
        if (u == v) return fail(CHORDAL_EPARSE, lineno, "self-loop at vertex " + uc);
        const long long lo = u < v ? u : v, hi = u < v ? v : u;
        uint8_t *rl = rows_out + (lo - 1) * row_bytes;
        const long long hb = hi - 1, lbit = lo - 1;
        if ((rl[hb >> 3] >> (hb & 7)) & 1)
            return fail(CHORDAL_EPARSE, lineno,
                        "duplicate edge (" + std::to_string(lo) + ", " + std::to_string(hi) + ")");
        ++edges_seen;
        if (edges_seen > m) return fail(CHORDAL_EPARSE, lineno, "more than the declared " + m_canon + " edges");
        rl[hb >> 3] |= (uint8_t)(1u << (hb & 7));
        rows_out[hb * row_bytes + (lbit >> 3)] |= (uint8_t)(1u << (lbit & 7));
    }
    if (n < 0) return fail(CHORDAL_EPARSE, -1, "missing header 'p <n> <m>'");
    if (edges_seen != m)
        return fail(CHORDAL_EPARSE, header_line,
                    "header declares " + m_canon + " edges but " + std::to_string(edges_seen) + " found");
    *n_out = n;
    *m_out = edges_seen;
    return CHORDAL_OK;
}

int64_t chordal_write_graph_text(const uint8_t *rows, int64_t n, int64_t row_bytes, int64_t m, char *out,
                                 int64_t out_cap) {
    // "p n m\n" then "e u v\n" for u < v ascending; returns the byte count
    // (the size needed when out is NULL or too small), or -1 on bad arguments.
    if (n < 0 || (n > 0 && (!rows || row_bytes < (n + 7) / 8))) return -1;
    auto ndig = [](long long x) { int d = 1; while (x >= 10) { x /= 10; ++d; } return d; };
    auto put = [](char *o, long long x, int d) { for (int k = d - 1; k >= 0; --k) { o[k] = (char)('0' + x % 10); x /= 10; } };
    const std::string head = "p " + std::to_string(n) + " " + std::to_string(m) + "\n";
    // size: "e " + digits(u) + " " + digits(v) + "\n" per edge u < v
    int64_t size = (int64_t)head.size();
    std::vector<int> dig((size_t)n + 1);
    for (int64_t v = 1; v <= n; ++v) dig[v] = ndig(v);
    std::vector<int64_t> rowsize((size_t)n, 0);
    for (int64_t u = 0; u < n; ++u) {
        const uint8_t *r = rows + u * row_bytes;
        int64_t sz = 0, cnt = 0;
        for (int64_t w = (u + 1) >> 3; w < (n + 7) >> 3; ++w) {
            unsigned byte = r[w];
            if (w == ((u + 1) >> 3)) byte &= 0xFFu << ((u + 1) & 7);
            while (byte) {
                const int64_t v = 8 * w + __builtin_ctz(byte);
                byte &= byte - 1;
                if (v >= n) break;
                sz += dig[v + 1];
                ++cnt;
            }
        }
        rowsize[u] = sz + cnt * (4 + dig[u + 1]);
        size += rowsize[u];
    }
    if (!out || out_cap < size) return size;
    memcpy(out, head.data(), head.size());
    char *o = out + head.size();
    for (int64_t u = 0; u < n; ++u) {
        if (!rowsize[u]) continue;
        const uint8_t *r = rows + u * row_bytes;
        const int du = dig[u + 1];
        char ub[24];
        put(ub, u + 1, du);
        for (int64_t w = (u + 1) >> 3; w < (n + 7) >> 3; ++w) {
            unsigned byte = r[w];
            if (w == ((u + 1) >> 3)) byte &= 0xFFu << ((u + 1) & 7);
            while (byte) {
                const int64_t v = 8 * w + __builtin_ctz(byte);
                byte &= byte - 1;
                if (v >= n) break;
                *o++ = 'e';
                *o++ = ' ';
                memcpy(o, ub, (size_t)du);
                o += du;
                *o++ = ' ';
                put(o, v + 1, dig[v + 1]);
                o += dig[v + 1];
                *o++ = '\n';
            }
        }
    }
    return size;
}

int chordal_parse_ordering_text(const char *text, int64_t len, int64_t n, int64_t *order_out, int64_t *count_out,
                                int64_t *err_line, char *err_msg, int64_t err_cap) {
    // text.split() then int() of every field (textio.py:96-106).  Writes up to n
    // values; *count_out = the number of fields.  A non-integer field fails with
    // ParseError("ordering entries must be integers: invalid literal for int()
    // with base 10: '<field>'"); the caller checks the count (InvalidOrdering).
    if (len < 0 || (len > 0 && !text) || !count_out) return CHORDAL_EINVAL;
    const unsigned char *p = reinterpret_cast<const unsigned char *>(text), *end = p + len;
    Err er;
    for (const unsigned char *q = p; q < end;) {
        if (*q < 0x80) { ++q; continue; }
        const int k = utf8_len(q, end);
        if (!k) {
            er.status = CHORDAL_EUTF8;
            er.msg = "input is not valid UTF-8";
            put_err(er, err_line, err_msg, err_cap);
            return CHORDAL_EUTF8;
        }
        q += k;
    }
    int64_t count = 0;
    std::string canon;
    while (p < end) {
        int s;
        while (p < end && ((s = space_at(p, end)) > 0 || (s = line_break(p, end)) > 0)) p += s;
        if (p >= end) break;
        const unsigned char *fb = p;
        while (p < end && space_at(p, end) == 0 && line_break(p, end) == 0)
            p += (*p < 0x80) ? 1 : utf8_len(p, end);
        long long v;
        bool big;
        if (!parse_int(Field{fb, p}, canon, v, big)) {
            er.status = CHORDAL_EPARSE;
            er.msg = "ordering entries must be integers: invalid literal for int() with base 10: '" +
                     std::string(reinterpret_cast<const char *>(fb), p - fb) + "'";
            put_err(er, err_line, err_msg, err_cap);
            return CHORDAL_EPARSE;
        }
        if (order_out && count < n) order_out[count] = big ? (v < 0 ? INT64_MIN : INT64_MAX) : v;
        ++count;
    }
    *count_out = count;
    return CHORDAL_OK;
}

}  // extern "C"
