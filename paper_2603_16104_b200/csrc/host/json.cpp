// JSON reader / writer of csrc/host/json.hpp.
#include "json.hpp"

#include <cctype>
#include <cstdio>

namespace hk::json {

namespace {

class Parser {
  public:
    explicit Parser(const std::string& s) : s_(s) {}
    Value doc() {
        Value v = value();
        ws();
        if (p_ != s_.size()) err("unexpected trailing characters");
        return v;
    }

  private:
    [[noreturn]] void err(const std::string& what) const {
        throw std::runtime_error("parse error at byte " + std::to_string(p_) + ": " + what);
    }
    void ws() {
        while (p_ < s_.size() && (s_[p_] == ' ' || s_[p_] == '\t' || s_[p_] == '\n' || s_[p_] == '\r')) ++p_;
    }
    bool lit(const char* w) {
        const std::size_t n = std::char_traits<char>::length(w);
        if (s_.compare(p_, n, w) == 0) {
            p_ += n;
            return true;
        }
        return false;
    }
    static void utf8(std::string& out, unsigned cp) {
        if (cp < 0x80) {
            out.push_back(static_cast<char>(cp));
        } else if (cp < 0x800) {
            out.push_back(static_cast<char>(0xC0 | (cp >> 6)));
            out.push_back(static_cast<char>(0x80 | (cp & 0x3F)));
        } else if (cp < 0x10000) {
            out.push_back(static_cast<char>(0xE0 | (cp >> 12)));
            out.push_back(static_cast<char>(0x80 | ((cp >> 6) & 0x3F)));
            out.push_back(static_cast<char>(0x80 | (cp & 0x3F)));
        } else {
            out.push_back(static_cast<char>(0xF0 | (cp >> 18)));
            out.push_back(static_cast<char>(0x80 | ((cp >> 12) & 0x3F)));
            out.push_back(static_cast<char>(0x80 | ((cp >> 6) & 0x3F)));
            out.push_back(static_cast<char>(0x80 | (cp & 0x3F)));
        }
    }
    unsigned hex4() {
        if (p_ + 4 > s_.size()) err("bad \\u escape");
        unsigned v = 0;
        for (int k = 0; k < 4; ++k) {
            const char c = s_[p_++];
            v <<= 4;
            if (c >= '0' && c <= '9') v |= static_cast<unsigned>(c - '0');
            else if (c >= 'a' && c <= 'f') v |= static_cast<unsigned>(c - 'a' + 10);
            else if (c >= 'A' && c <= 'F') v |= static_cast<unsigned>(c - 'A' + 10);
            else err("bad \\u escape");
        }
        return v;
    }
    std::string string() {
        ++p_;  // opening quote
        std::string out;
        while (true) {
            if (p_ >= s_.size()) err("unterminated string");
            const char c = s_[p_++];
            if (c == '"') return out;
            if (static_cast<unsigned char>(c) < 0x20) err("control character in string");
            if (c != '\\') {
                out.push_back(c);
                continue;
            }
            if (p_ >= s_.size()) err("unterminated string");
            const char e = s_[p_++];
            switch (e) {
                case '"': out.push_back('"'); break;
                case '\\': out.push_back('\\'); break;
                case '/': out.push_back('/'); break;
                case 'b': out.push_back('\b'); break;
                case 'f': out.push_back('\f'); break;
                case 'n': out.push_back('\n'); break;
                case 'r': out.push_back('\r'); break;
                case 't': out.push_back('\t'); break;
                case 'u': {
                    unsigned cp = hex4();
                    if (cp >= 0xD800 && cp <= 0xDBFF && s_.compare(p_, 2, "\\u") == 0) {
                        p_ += 2;
                        const unsigned lo = hex4();
                        cp = 0x10000 + ((cp - 0xD800) << 10) + (lo - 0xDC00);
                    }
                    utf8(out, cp);
                    break;
                }
                default: err("bad escape");
            }
        }
    }
    Value number() {
        const std::size_t st = p_;
        bool neg = false, frac = false;
        if (s_[p_] == '-') {
            neg = true;
            ++p_;
        }
        if (p_ >= s_.size() || !std::isdigit(static_cast<unsigned char>(s_[p_]))) err("bad number");
        while (p_ < s_.size() && std::isdigit(static_cast<unsigned char>(s_[p_]))) ++p_;
        if (p_ < s_.size() && s_[p_] == '.') {
            frac = true;
            ++p_;
            if (p_ >= s_.size() || !std::isdigit(static_cast<unsigned char>(s_[p_]))) err("bad number");
            while (p_ < s_.size() && std::isdigit(static_cast<unsigned char>(s_[p_]))) ++p_;
        }
        if (p_ < s_.size() && (s_[p_] == 'e' || s_[p_] == 'E')) {
            frac = true;
            ++p_;
            if (p_ < s_.size() && (s_[p_] == '+' || s_[p_] == '-')) ++p_;
            if (p_ >= s_.size() || !std::isdigit(static_cast<unsigned char>(s_[p_]))) err("bad number");
            while (p_ < s_.size() && std::isdigit(static_cast<unsigned char>(s_[p_]))) ++p_;
        }
        const char* b = s_.data() + st;
        const char* e = s_.data() + p_;
        if (!frac) {
            if (neg) {
                std::int64_t v = 0;
                if (std::from_chars(b, e, v).ec == std::errc()) return Value::sint(v);
            } else {
                std::uint64_t v = 0;
                if (std::from_chars(b, e, v).ec == std::errc()) return Value::uint(v);
            }
        }
        double d = 0;
        if (std::from_chars(b, e, d).ec != std::errc()) err("bad number");
        return Value::dbl(d);
    }
    Value value() {
        ws();
        if (p_ >= s_.size()) err("unexpected end of input");
        const char c = s_[p_];
        if (c == '{') {
            ++p_;
            Value v = Value::object();
            ws();
            if (p_ < s_.size() && s_[p_] == '}') {
                ++p_;
                return v;
            }
            while (true) {
                ws();
                if (p_ >= s_.size() || s_[p_] != '"') err("expected a string key");
                std::string k = string();
                ws();
                if (p_ >= s_.size() || s_[p_] != ':') err("expected ':'");
                ++p_;
                v.obj[k] = value();
                ws();
                if (p_ < s_.size() && s_[p_] == ',') {
                    ++p_;
                    continue;
                }
                if (p_ < s_.size() && s_[p_] == '}') {
                    ++p_;
                    return v;
                }
                err("expected ',' or '}'");
            }
        }
        if (c == '[') {
            ++p_;
            Value v = Value::array();
            ws();
            if (p_ < s_.size() && s_[p_] == ']') {
                ++p_;
                return v;
            }
            while (true) {
                v.arr.push_back(value());
                ws();
                if (p_ < s_.size() && s_[p_] == ',') {
                    ++p_;
                    continue;
                }
                if (p_ < s_.size() && s_[p_] == ']') {
                    ++p_;
                    return v;
                }
                err("expected ',' or ']'");
            }
        }
        if (c == '"') return Value::str(string());
        if (lit("true")) return Value::boolean(true);
        if (lit("false")) return Value::boolean(false);
        if (lit("null")) return Value();
        return number();
    }
    const std::string& s_;
    std::size_t p_ = 0;
};

void escape(std::string& o, const std::string& s) {
    o.push_back('"');
    for (const char ch : s) {
        const auto c = static_cast<unsigned char>(ch);
        switch (ch) {
            case '"': o += "\\\""; break;
            case '\\': o += "\\\\"; break;
            case '\b': o += "\\b"; break;
            case '\f': o += "\\f"; break;
            case '\n': o += "\\n"; break;
            case '\r': o += "\\r"; break;
            case '\t': o += "\\t"; break;
            default:
                if (c < 0x20) {
                    char buf[8];
                    std::snprintf(buf, sizeof(buf), "\\u%04x", c);
                    o += buf;
                } else {
                    o.push_back(ch);
                }
        }
    }
    o.push_back('"');
}

void number(std::string& o, double d) {
    if (!std::isfinite(d)) {
        o += "null";
        return;
    }
    char buf[64];
    const auto r = std::to_chars(buf, buf + sizeof(buf), d);
    std::string t(buf, r.ptr);
    if (t.find_first_of(".e") == std::string::npos) t += ".0";
    o += t;
}

bool scalar(const Value& v) { return v.kind != Value::kArray && v.kind != Value::kObject; }

void write(std::string& o, const Value& v, int indent, int level) {
    const std::string pad(static_cast<std::size_t>(indent * (level + 1)), ' ');
    const std::string close(static_cast<std::size_t>(indent * level), ' ');
    switch (v.kind) {
        case Value::kNull: o += "null"; break;
        case Value::kBool: o += v.b ? "true" : "false"; break;
        case Value::kInt: o += std::to_string(v.i); break;
        case Value::kUInt: o += std::to_string(v.u); break;
        case Value::kDouble: number(o, v.d); break;
        case Value::kString: escape(o, v.s); break;
        case Value::kArray: {
            if (v.arr.empty()) {
                o += "[]";
                break;
            }
            bool flat = true;
            for (const Value& e : v.arr) flat = flat && scalar(e);
            if (flat) {  // the reference build prints arrays of scalars on one line
                o.push_back('[');
                for (std::size_t k = 0; k < v.arr.size(); ++k) {
                    if (k) o.push_back(',');
                    write(o, v.arr[k], indent, level + 1);
                }
                o.push_back(']');
                break;
            }
            o += "[\n";
            for (std::size_t k = 0; k < v.arr.size(); ++k) {
                o += pad;
                write(o, v.arr[k], indent, level + 1);
                o += k + 1 < v.arr.size() ? ",\n" : "\n";
            }
            o += close + "]";
            break;
        }
        case Value::kObject: {
            if (v.obj.empty()) {
                o += "{}";
                break;
            }
            o += "{\n";
            std::size_t k = 0;
            for (const auto& [key, e] : v.obj) {
                o += pad;
                escape(o, key);
                o += ": ";
                write(o, e, indent, level + 1);
                o += ++k < v.obj.size() ? ",\n" : "\n";
            }
            o += close + "}";
            break;
        }
    }
}

}  // namespace

Value parse(const std::string& text) { return Parser(text).doc(); }

std::string dump(const Value& v, int indent) {
    std::string o;
    write(o, v, indent, 0);
    return o;
}

std::int64_t Value::as_int() const {
    if (kind == kInt) return i;
    if (kind == kUInt) {
        if (u > static_cast<std::uint64_t>(INT64_MAX)) throw std::runtime_error("json: integer out of range");
        return static_cast<std::int64_t>(u);
    }
    if (kind == kDouble && std::floor(d) == d) return static_cast<std::int64_t>(d);
    throw std::runtime_error("json: type must be number");
}
std::uint64_t Value::as_uint() const {
    if (kind == kUInt) return u;
    if (kind == kInt) {
        if (i < 0) throw std::runtime_error("json: negative value for an unsigned field");
        return static_cast<std::uint64_t>(i);
    }
    if (kind == kDouble && d >= 0 && std::floor(d) == d) return static_cast<std::uint64_t>(d);
    throw std::runtime_error("json: type must be number");
}
double Value::as_double() const {
    if (kind == kDouble) return d;
    if (kind == kUInt) return static_cast<double>(u);
    if (kind == kInt) return static_cast<double>(i);
    throw std::runtime_error("json: type must be number");
}
const std::string& Value::as_string() const {
    if (kind != kString) throw std::runtime_error("json: type must be string");
    return s;
}
bool Value::as_bool() const {
    if (kind != kBool) throw std::runtime_error("json: type must be boolean");
    return b;
}

}  // namespace hk::json
