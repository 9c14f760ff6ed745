// json_lite.cpp — see json_lite.h.
#include "json_lite.h"

#include <algorithm>
#include <charconv>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>

namespace json_lite {

Value Value::integer(int64_t v) {
    Value x;
    x.kind_ = Kind::integer;
    x.i_ = v;
    return x;
}
Value Value::boolean(bool v) {
    Value x;
    x.kind_ = Kind::boolean;
    x.b_ = v;
    return x;
}
Value Value::real(double v) {
    Value x;
    x.kind_ = Kind::real;
    x.d_ = v;
    return x;
}
Value Value::str(std::string v) {
    Value x;
    x.kind_ = Kind::string;
    x.s_ = std::move(v);
    return x;
}
Value Value::array() {
    Value x;
    x.kind_ = Kind::array;
    return x;
}
Value Value::object() {
    Value x;
    x.kind_ = Kind::object;
    return x;
}

int64_t Value::as_int() const {
    if (kind_ == Kind::integer)
        return i_;
    if (kind_ == Kind::real && std::isfinite(d_) && std::trunc(d_) == d_ && std::fabs(d_) < 9.2e18)
        return static_cast<int64_t>(d_);
    throw TypeError("expected an integer");
}
double Value::as_double() const {
    if (kind_ == Kind::integer)
        return static_cast<double>(i_);
    if (kind_ == Kind::real)
        return d_;
    throw TypeError("expected a number");
}
const std::string& Value::as_string() const {
    if (kind_ != Kind::string)
        throw TypeError("expected a string");
    return s_;
}
const std::vector<Value>& Value::items() const {
    if (kind_ != Kind::array)
        throw TypeError("expected an array");
    return a_;
}
const Value& Value::at(const std::string& key) const {
    if (kind_ != Kind::object)
        throw TypeError("expected an object");
    auto it = o_.find(key);
    if (it == o_.end())
        throw TypeError("missing key '" + key + "'");
    return it->second;
}
bool Value::has(const std::string& key) const { return kind_ == Kind::object && o_.count(key) != 0; }
void Value::push(Value v) {
    if (kind_ != Kind::array)
        throw TypeError("push on a non-array");
    a_.push_back(std::move(v));
}
void Value::set(const std::string& key, Value v) {
    if (kind_ != Kind::object)
        throw TypeError("set on a non-object");
    o_[key] = std::move(v);
}

namespace {

void put_string(std::string& out, const std::string& s) {
    out += '"';
    for (unsigned char c : s) {
        switch (c) {
        case '"': out += "\\\""; break;
        case '\\': out += "\\\\"; break;
        case '\b': out += "\\b"; break;
        case '\f': out += "\\f"; break;
        case '\n': out += "\\n"; break;
        case '\r': out += "\\r"; break;
        case '\t': out += "\\t"; break;
        default:
            if (c < 0x20) {
                char buf[8];
                std::snprintf(buf, sizeof buf, "\\u%04x", c);
                out += buf;
            } else {
                out += static_cast<char>(c);
            }
        }
    }
    out += '"';
}

// Shortest round-trip digits of v laid out like nlohmann::json's dtoa
// (decimal for -4 < e10 <= 15, else scientific with a signed 2+ digit
// exponent; integral values keep a trailing ".0").
void put_double(std::string& out, double v) {
    if (!std::isfinite(v)) {
        out += "null";
        return;
    }
    if (v == 0.0) {
        out += std::signbit(v) ? "-0.0" : "0.0";
        return;
    }
    char buf[64];
    auto r = std::to_chars(buf, buf + sizeof buf, v, std::chars_format::scientific);
    std::string sci(buf, r.ptr);  // [-]d[.ddd]e[+-]XX
    std::string sign;
    if (sci[0] == '-') {
        sign = "-";
        sci.erase(0, 1);
    }
    const size_t epos = sci.find('e');
    std::string digits = sci.substr(0, epos);
    digits.erase(std::remove(digits.begin(), digits.end(), '.'), digits.end());
    const int exp10 = std::atoi(sci.c_str() + epos + 1);
    const int k = static_cast<int>(digits.size());
    const int n = exp10 + 1;  // decimal point position relative to the digit string
    std::string s;
    if (k <= n && n <= 15) {
        s = digits + std::string(static_cast<size_t>(n - k), '0') + ".0";
    } else if (0 < n && n <= 15) {
        s = digits.substr(0, static_cast<size_t>(n)) + "." + digits.substr(static_cast<size_t>(n));
    } else if (-4 < n && n <= 0) {
        s = "0." + std::string(static_cast<size_t>(-n), '0') + digits;
    } else {
        s = digits.substr(0, 1);
        if (k > 1)
            s += "." + digits.substr(1);
        const int e = n - 1;
        char eb[16];
        std::snprintf(eb, sizeof eb, "e%c%02d", e < 0 ? '-' : '+', e < 0 ? -e : e);
        s += eb;
    }
    out += sign + s;
}

struct Parser {
    const std::string& t;
    size_t p = 0;

    [[noreturn]] void error(const std::string& what) const {
        throw ParseError(what + " at offset " + std::to_string(p));
    }
    void ws() {
        while (p < t.size() && (t[p] == ' ' || t[p] == '\t' || t[p] == '\n' || t[p] == '\r'))
            ++p;
    }
    bool eat(char c) {
        ws();
        if (p < t.size() && t[p] == c) {
            ++p;
            return true;
        }
        return false;
    }
    void expect_word(const char* w) {
        const size_t n = std::strlen(w);
        if (t.compare(p, n, w) != 0)
            error("invalid literal");
        p += n;
    }
    static void utf8(std::string& out, uint32_t cp) {
        if (cp < 0x80) {
            out += static_cast<char>(cp);
        } else if (cp < 0x800) {
            out += static_cast<char>(0xC0 | (cp >> 6));
            out += static_cast<char>(0x80 | (cp & 0x3F));
        } else if (cp < 0x10000) {
            out += static_cast<char>(0xE0 | (cp >> 12));
            out += static_cast<char>(0x80 | ((cp >> 6) & 0x3F));
            out += static_cast<char>(0x80 | (cp & 0x3F));
        } else {
            out += static_cast<char>(0xF0 | (cp >> 18));
            out += static_cast<char>(0x80 | ((cp >> 12) & 0x3F));
            out += static_cast<char>(0x80 | ((cp >> 6) & 0x3F));
            out += static_cast<char>(0x80 | (cp & 0x3F));
        }
    }
    uint32_t hex4() {
        if (p + 4 > t.size())
            error("truncated \\u escape");
        uint32_t v = 0;
        for (int i = 0; i < 4; ++i) {
            const char c = t[p++];
            v <<= 4;
            if (c >= '0' && c <= '9')
                v |= static_cast<uint32_t>(c - '0');
            else if (c >= 'a' && c <= 'f')
                v |= static_cast<uint32_t>(c - 'a' + 10);
            else if (c >= 'A' && c <= 'F')
                v |= static_cast<uint32_t>(c - 'A' + 10);
            else
                error("bad \\u escape");
        }
        return v;
    }
    std::string string() {
        // at the opening quote
        ++p;
        std::string s;
        while (true) {
            if (p >= t.size())
                error("unterminated string");
            const char c = t[p++];
            if (c == '"')
                return s;
            if (static_cast<unsigned char>(c) < 0x20)
                error("control character in string");
            if (c != '\\') {
                s += c;
                continue;
            }
            if (p >= t.size())
                error("unterminated escape");
            const char e = t[p++];
            switch (e) {
            case '"': s += '"'; break;
            case '\\': s += '\\'; break;
            case '/': s += '/'; break;
            case 'b': s += '\b'; break;
            case 'f': s += '\f'; break;
            case 'n': s += '\n'; break;
            case 'r': s += '\r'; break;
            case 't': s += '\t'; break;
            case 'u': {
                uint32_t cp = hex4();
                if (cp >= 0xD800 && cp < 0xDC00) {
                    if (t.compare(p, 2, "\\u") != 0)
                        error("lone surrogate");
                    p += 2;
                    const uint32_t lo = hex4();
                    if (lo < 0xDC00 || lo >= 0xE000)
                        error("bad surrogate pair");
                    cp = 0x10000 + ((cp - 0xD800) << 10) + (lo - 0xDC00);
                }
                utf8(s, cp);
                break;
            }
            default:
                error("bad escape");
            }
        }
    }
    Value number() {
        const size_t b = p;
        if (t[p] == '-')
            ++p;
        auto digits = [&] {
            const size_t s = p;
            while (p < t.size() && t[p] >= '0' && t[p] <= '9')
                ++p;
            return p - s;
        };
        if (p < t.size() && t[p] == '0')
            ++p;
        else if (digits() == 0)
            error("bad number");
        bool integral = true;
        if (p < t.size() && t[p] == '.') {
            ++p;
            integral = false;
            if (digits() == 0)
                error("bad fraction");
        }
        if (p < t.size() && (t[p] == 'e' || t[p] == 'E')) {
            ++p;
            integral = false;
            if (p < t.size() && (t[p] == '+' || t[p] == '-'))
                ++p;
            if (digits() == 0)
                error("bad exponent");
        }
        const std::string tok = t.substr(b, p - b);
        if (integral) {
            int64_t v = 0;
            auto r = std::from_chars(tok.data(), tok.data() + tok.size(), v);
            if (r.ec == std::errc())
                return Value::integer(v);
        }
        return Value::real(std::strtod(tok.c_str(), nullptr));
    }
    Value value(int depth) {
        if (depth > 512)
            error("nesting too deep");
        ws();
        if (p >= t.size())
            error("unexpected end of input");
        const char c = t[p];
        if (c == '{') {
            ++p;
            Value o = Value::object();
            if (eat('}'))
                return o;
            do {
                ws();
                if (p >= t.size() || t[p] != '"')
                    error("expected a key");
                std::string k = string();
                if (!eat(':'))
                    error("expected ':'");
                o.set(k, value(depth + 1));
            } while (eat(','));
            if (!eat('}'))
                error("expected '}'");
            return o;
        }
        if (c == '[') {
            ++p;
            Value a = Value::array();
            if (eat(']'))
                return a;
            do {
                a.push(value(depth + 1));
            } while (eat(','));
            if (!eat(']'))
                error("expected ']'");
            return a;
        }
        if (c == '"')
            return Value::str(string());
        if (c == 't') {
            expect_word("true");
            return Value::boolean(true);
        }
        if (c == 'f') {
            expect_word("false");
            return Value::boolean(false);
        }
        if (c == 'n') {
            expect_word("null");
            return Value();
        }
        if (c == '-' || (c >= '0' && c <= '9'))
            return number();
        error("unexpected character");
    }
};

}  // namespace

void Value::dump_to(std::string& out, int indent, int depth) const {
    const std::string pad(static_cast<size_t>(indent * (depth + 1)), ' ');
    const std::string pad0(static_cast<size_t>(indent * depth), ' ');
    switch (kind_) {
    case Kind::null: out += "null"; break;
    case Kind::boolean: out += b_ ? "true" : "false"; break;
    case Kind::integer: out += std::to_string(i_); break;
    case Kind::real: put_double(out, d_); break;
    case Kind::string: put_string(out, s_); break;
    case Kind::array:
        if (a_.empty()) {
            out += "[]";
            break;
        }
        if (std::all_of(a_.begin(), a_.end(), [](const Value& v) {
                return v.kind_ != Kind::array && v.kind_ != Kind::object;
            })) {
            // arrays of scalars stay on one line, comma-separated without
            // spaces, as in the reference's plan files ("window_set": [14,21])
            out += "[";
            for (size_t i = 0; i < a_.size(); ++i) {
                a_[i].dump_to(out, indent, depth + 1);
                if (i + 1 < a_.size())
                    out += ",";
            }
            out += "]";
            break;
        }
        out += "[\n";
        for (size_t i = 0; i < a_.size(); ++i) {
            out += pad;
            a_[i].dump_to(out, indent, depth + 1);
            out += i + 1 < a_.size() ? ",\n" : "\n";
        }
        out += pad0 + "]";
        break;
    case Kind::object:
        if (o_.empty()) {
            out += "{}";
            break;
        }
        out += "{\n";
        {
            size_t i = 0;
            for (const auto& [k, v] : o_) {
                out += pad;
                put_string(out, k);
                out += ": ";
                v.dump_to(out, indent, depth + 1);
                out += ++i < o_.size() ? ",\n" : "\n";
            }
        }
        out += pad0 + "}";
        break;
    }
}

std::string Value::dump(int indent) const {
    std::string out;
    dump_to(out, indent, 0);
    return out;
}

Value parse(const std::string& text) {
    Parser ps{text};
    Value v = ps.value(0);
    ps.ws();
    if (ps.p != text.size())
        ps.error("trailing characters");
    return v;
}

}  // namespace json_lite
