// TEST INFRASTRUCTURE ONLY — never linked into the product library.
//
// nlohmann/json is not installed in this image. The reference's dataio.cpp
// (load_dataset / write_dataset, dataio.cpp:116-254) uses a small slice of the
// nlohmann::json API for meta.json; this header implements that slice so
// dataio.cpp compiles unmodified into oracle/_ref (oracle/Makefile) and the
// dataset files the reference writes can be produced and read here:
//   json::array({...}), operator[](key), at(key) / at(index), value(key, default),
//   contains(key), push_back, range-for over arrays, implicit conversion to
//   arithmetic types and std::string, dump(indent), operator>>(istream, json).
// The serialisation follows nlohmann::json's documented defaults: objects are
// std::map-ordered (keys sorted), dump(2) puts every array/object element on its
// own line, and doubles print as the shortest round-trip digits in the layout of
// nlohmann's dtoa format_buffer (integral values end in ".0", exponent form
// outside [1e-5, 1e15), at least two exponent digits).
#pragma once

#include <cctype>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <initializer_list>
#include <istream>
#include <iterator>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <vector>

namespace nlohmann {

class json {
public:
    enum class kind { null, boolean, integer, number, string, array, object };

    json() = default;
    json(std::nullptr_t) {}
    json(bool b) : k_(kind::boolean), b_(b) {}
    template <typename T, typename std::enable_if<std::is_integral<T>::value && !std::is_same<T, bool>::value,
                                                  int>::type = 0>
    json(T i) : k_(kind::integer), i_(static_cast<std::int64_t>(i)) {}
    template <typename T, typename std::enable_if<std::is_floating_point<T>::value, int>::type = 0>
    json(T d) : k_(kind::number), d_(static_cast<double>(d)) {}
    json(const std::string& s) : k_(kind::string), s_(s) {}
    json(const char* s) : k_(kind::string), s_(s) {}

    static json array(std::initializer_list<json> items = {}) {
        json j;
        j.k_ = kind::array;
        j.a_.assign(items.begin(), items.end());
        return j;
    }
    static json object() {
        json j;
        j.k_ = kind::object;
        return j;
    }

    // ---- access
    json& operator[](const std::string& key) {
        if (k_ == kind::null) k_ = kind::object;
        if (k_ != kind::object) throw std::domain_error("json: operator[] with a key on a non-object");
        return o_[key];
    }
    const json& at(const std::string& key) const {
        if (k_ != kind::object) throw std::domain_error("json: at(key) on a non-object");
        auto it = o_.find(key);
        if (it == o_.end()) throw std::out_of_range("json: key '" + key + "' not found");
        return it->second;
    }
    const json& at(std::size_t i) const {
        if (k_ != kind::array) throw std::domain_error("json: at(index) on a non-array");
        if (i >= a_.size()) throw std::out_of_range("json: array index out of range");
        return a_[i];
    }
    bool contains(const std::string& key) const { return k_ == kind::object && o_.count(key) > 0; }
    std::string value(const std::string& key, const char* def) const {
        return contains(key) ? at(key).get_string() : std::string(def);
    }
    void push_back(const json& v) {
        if (k_ == kind::null) k_ = kind::array;
        if (k_ != kind::array) throw std::domain_error("json: push_back on a non-array");
        a_.push_back(v);
    }
    std::vector<json>::const_iterator begin() const { return a_.begin(); }
    std::vector<json>::const_iterator end() const { return a_.end(); }

    // ---- conversions (nlohmann's implicit get<T>())
    template <typename T, typename std::enable_if<std::is_arithmetic<T>::value, int>::type = 0>
    operator T() const {
        if (k_ == kind::integer) return static_cast<T>(i_);
        if (k_ == kind::number) return static_cast<T>(d_);
        if (k_ == kind::boolean) return static_cast<T>(b_);
        throw std::domain_error("json: value is not a number");
    }
    operator std::string() const { return get_string(); }
    const std::string& get_string() const {
        if (k_ != kind::string) throw std::domain_error("json: value is not a string");
        return s_;
    }

    // ---- serialisation
    std::string dump(int indent = -1) const {
        std::string out;
        write(out, indent, 0);
        return out;
    }
    friend std::istream& operator>>(std::istream& in, json& j) {
        std::string text((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
        std::size_t p = 0;
        j = parse_value(text, p);
        skip_ws(text, p);
        if (p != text.size()) throw std::invalid_argument("json: parse error: trailing characters");
        return in;
    }

private:
    kind k_ = kind::null;
    bool b_ = false;
    std::int64_t i_ = 0;
    double d_ = 0.0;
    std::string s_;
    std::vector<json> a_;
    std::map<std::string, json> o_;

    static void put_number(std::string& out, double x) {
        if (!(x == x) || x == 1.0 / 0.0 || x == -1.0 / 0.0) {
            out += "null";  // nlohmann writes non-finite numbers as null
            return;
        }
        if (x == 0.0) {
            out += std::signbit(x) ? "-0.0" : "0.0";
            return;
        }
        // shortest %e digits that round-trip
        char buf[64];
        int prec = 0;
        for (prec = 0; prec < 17; ++prec) {
            std::snprintf(buf, sizeof buf, "%.*e", prec, x);
            if (std::strtod(buf, nullptr) == x) break;
        }
        // split "[-]d.ddde[+-]XX" into digits and the decimal point position n
        std::string s(buf);
        std::string sign;
        if (s[0] == '-') {
            sign = "-";
            s = s.substr(1);
        }
        const std::size_t e = s.find('e');
        std::string digits = s.substr(0, 1) + (e > 2 ? s.substr(2, e - 2) : std::string());
        while (digits.size() > 1 && digits.back() == '0') digits.pop_back();
        const int exp10 = std::atoi(s.c_str() + e + 1);
        const int k = int(digits.size());
        const int n = exp10 + 1;  // value = 0.d1..dk * 10^n
        std::string r;
        if (k <= n && n <= 15) {
            r = digits + std::string(std::size_t(n - k), '0') + ".0";
        } else if (0 < n && n <= 15) {
            r = digits.substr(0, std::size_t(n)) + "." + digits.substr(std::size_t(n));
        } else if (-4 < n && n <= 0) {
            r = "0." + std::string(std::size_t(-n), '0') + digits;
        } else {
            r = digits.substr(0, 1);
            if (k > 1) r += "." + digits.substr(1);
            const int ex = n - 1;
            char eb[16];
            std::snprintf(eb, sizeof eb, "e%c%02d", ex < 0 ? '-' : '+', ex < 0 ? -ex : ex);
            r += eb;
        }
        out += sign + r;
    }
    static void put_string(std::string& out, const std::string& s) {
        out += '"';
        for (unsigned char c : s) {
            switch (c) {
                case '"': out += "\\\""; break;
                case '\\': out += "\\\\"; break;
                case '\n': out += "\\n"; break;
                case '\t': out += "\\t"; break;
                case '\r': out += "\\r"; break;
                case '\b': out += "\\b"; break;
                case '\f': out += "\\f"; break;
                default:
                    if (c < 0x20) {
                        char b[8];
                        std::snprintf(b, sizeof b, "\\u%04x", c);
                        out += b;
                    } else {
                        out += char(c);
                    }
            }
        }
        out += '"';
    }
    void write(std::string& out, int indent, int level) const {
        const bool pretty = indent >= 0;
        const std::string pad = pretty ? std::string(std::size_t(indent * (level + 1)), ' ') : "";
        const std::string pad_end = pretty ? std::string(std::size_t(indent * level), ' ') : "";
        switch (k_) {
            case kind::null: out += "null"; break;
            case kind::boolean: out += b_ ? "true" : "false"; break;
            case kind::integer: out += std::to_string(i_); break;
            case kind::number: put_number(out, d_); break;
            case kind::string: put_string(out, s_); break;
            case kind::array:
                if (a_.empty()) {
                    out += "[]";
                    break;
                }
                out += pretty ? "[\n" : "[";
                for (std::size_t i = 0; i < a_.size(); ++i) {
                    out += pad;
                    a_[i].write(out, indent, level + 1);
                    if (i + 1 < a_.size()) out += pretty ? ",\n" : ",";
                }
                out += pretty ? "\n" + pad_end + "]" : "]";
                break;
            case kind::object: {
                if (o_.empty()) {
                    out += "{}";
                    break;
                }
                out += pretty ? "{\n" : "{";
                std::size_t i = 0;
                for (const auto& kv : o_) {
                    out += pad;
                    put_string(out, kv.first);
                    out += pretty ? ": " : ":";
                    kv.second.write(out, indent, level + 1);
                    if (++i < o_.size()) out += pretty ? ",\n" : ",";
                }
                out += pretty ? "\n" + pad_end + "}" : "}";
                break;
            }
        }
    }

    // ---- parser (RFC 8259 subset: no \u escapes beyond ASCII)
    static void skip_ws(const std::string& t, std::size_t& p) {
        while (p < t.size() && (t[p] == ' ' || t[p] == '\n' || t[p] == '\r' || t[p] == '\t')) ++p;
    }
    [[noreturn]] static void fail(const char* what) {
        throw std::invalid_argument(std::string("json: parse error: ") + what);
    }
    static std::string parse_string(const std::string& t, std::size_t& p) {
        if (t[p] != '"') fail("expected string");
        ++p;
        std::string s;
        while (p < t.size() && t[p] != '"') {
            char c = t[p++];
            if (c == '\\') {
                if (p >= t.size()) fail("bad escape");
                const char e = t[p++];
                switch (e) {
                    case 'n': s += '\n'; break;
                    case 't': s += '\t'; break;
                    case 'r': s += '\r'; break;
                    case 'b': s += '\b'; break;
                    case 'f': s += '\f'; break;
                    case 'u': {
                        if (p + 4 > t.size()) fail("bad \\u escape");
                        const long cp = std::strtol(t.substr(p, 4).c_str(), nullptr, 16);
                        if (cp > 0x7f) fail("non-ASCII \\u escape");
                        s += char(cp);
                        p += 4;
                        break;
                    }
                    default: s += e;
                }
            } else {
                s += c;
            }
        }
        if (p >= t.size()) fail("unterminated string");
        ++p;
        return s;
    }
    static json parse_value(const std::string& t, std::size_t& p) {
        skip_ws(t, p);
        if (p >= t.size()) fail("unexpected end of input");
        const char c = t[p];
        if (c == '{') {
            json j = object();
            ++p;
            skip_ws(t, p);
            if (p < t.size() && t[p] == '}') {
                ++p;
                return j;
            }
            for (;;) {
                skip_ws(t, p);
                const std::string key = parse_string(t, p);
                skip_ws(t, p);
                if (p >= t.size() || t[p] != ':') fail("expected ':'");
                ++p;
                j.o_[key] = parse_value(t, p);
                skip_ws(t, p);
                if (p < t.size() && t[p] == ',') {
                    ++p;
                    continue;
                }
                if (p < t.size() && t[p] == '}') {
                    ++p;
                    return j;
                }
                fail("expected ',' or '}'");
            }
        }
        if (c == '[') {
            json j = array();
            ++p;
            skip_ws(t, p);
            if (p < t.size() && t[p] == ']') {
                ++p;
                return j;
            }
            for (;;) {
                j.a_.push_back(parse_value(t, p));
                skip_ws(t, p);
                if (p < t.size() && t[p] == ',') {
                    ++p;
                    continue;
                }
                if (p < t.size() && t[p] == ']') {
                    ++p;
                    return j;
                }
                fail("expected ',' or ']'");
            }
        }
        if (c == '"') return json(parse_string(t, p));
        if (t.compare(p, 4, "true") == 0) {
            p += 4;
            return json(true);
        }
        if (t.compare(p, 5, "false") == 0) {
            p += 5;
            return json(false);
        }
        if (t.compare(p, 4, "null") == 0) {
            p += 4;
            return json();
        }
        // number: integer unless it has a fraction or exponent
        const std::size_t s0 = p;
        if (t[p] == '-') ++p;
        bool is_float = false;
        while (p < t.size() && (std::isdigit(static_cast<unsigned char>(t[p])) || t[p] == '.' || t[p] == 'e' ||
                                t[p] == 'E' || t[p] == '+' || t[p] == '-')) {
            if (t[p] == '.' || t[p] == 'e' || t[p] == 'E') is_float = true;
            ++p;
        }
        if (p == s0 || (p == s0 + 1 && t[s0] == '-')) fail("unexpected character");
        const std::string num = t.substr(s0, p - s0);
        char* endp = nullptr;
        if (is_float) {
            const double d = std::strtod(num.c_str(), &endp);
            if (*endp) fail("bad number");
            return json(d);
        }
        const long long i = std::strtoll(num.c_str(), &endp, 10);
        if (*endp) fail("bad number");
        return json(i);
    }
};

}  // namespace nlohmann
