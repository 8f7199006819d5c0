/* CPython fast path of render_frame / FramePipeline.submit: reads the
 * reference Scene's attributes (duck-typed, as model.pack_scene does) into
 * C arrays and calls rt_render_v1 / rt_render_async_v1 with the GIL released
 * -- the per-frame host work of the reference's _scene_args + _render_kernel
 * call (renderer.py:282-300, 331-349) without ctypes marshalling.
 *
 * Anything unexpected (a non-float32 skybox, a malformed body, more bodies
 * than fit) returns None: the caller then takes the generic ctypes path,
 * which raises the reference's errors.  The two C-ABI entry points are handed
 * over once as addresses (set_entry_points), so this module links against
 * nothing but Python. */
#define PY_SSIZE_T_CLEAN
#include <Python.h>
#include <stdint.h>

typedef int (*render_fn)(void *, uint32_t *, void *, int32_t, int32_t, const double *, double, double, double, int32_t,
                         const int32_t *, const double *, const double *, const double *, const double *,
                         const double *, double, const double *, double, double, const float *, int32_t, int32_t,
                         int32_t, int32_t, int32_t, int32_t, int32_t);
typedef int (*async_fn)(void *, int32_t, uint32_t *, int32_t, int32_t, const double *, double, double, double, int32_t,
                        const int32_t *, const double *, const double *, const double *, const double *,
                        const double *, double, const double *, double, double, const float *, int32_t, int32_t,
                        int32_t, int32_t, int32_t, int32_t);

static render_fn g_render = NULL;
static async_fn g_async = NULL;

#define MAX_BODIES 1024

typedef struct {
    int n;
    int32_t kinds[MAX_BODIES];
    double pos[3 * MAX_BODIES], size[MAX_BODIES], color[3 * MAX_BODIES], refl[MAX_BODIES];
    double light_pos[3], light_color[3], light_radius, ambient, max_refl;
    const float *sky;
    int32_t sky_w, sky_h, has_sky;
    Py_buffer sky_view;
    int have_view;
} Packed;

static float g_no_sky[3] = {0.f, 0.f, 0.f};
static __thread Packed g_packed;

/* attribute names, interned once (PyInit__pyfast) */
enum { A_BODIES, A_KIND, A_POSITION, A_SIZE, A_COLOR, A_REFLECTIVITY, A_LIGHT, A_RADIUS, A_AMBIENT, A_MAX_REFL,
       A_SKYBOX, A_TEXELS, A_WIDTH, A_HEIGHT, A_N };
static const char *const g_attr_names[A_N] = {"bodies", "kind",  "position",         "size",   "color",
                                              "reflectivity", "light", "radius", "ambient", "max_reflectivity",
                                              "skybox", "texels", "width", "height"};
static PyObject *g_attr[A_N];

static PyObject *get(PyObject *o, int a) { return PyObject_GetAttr(o, g_attr[a]); }

/* a float (or int) item without the generic number protocol when it is a float */
static inline int as_double(PyObject *v, double *out) {
    if (PyFloat_CheckExact(v)) {
        *out = PyFloat_AS_DOUBLE(v);
        return 1;
    }
    *out = PyFloat_AsDouble(v);
    if (*out == -1.0 && PyErr_Occurred()) {
        PyErr_Clear();
        return 0;
    }
    return 1;
}

/* 3 floats from a sequence attribute; 0 on failure (no Python error left set) */
static int vec3(PyObject *o, double *out) {
    if (PyTuple_CheckExact(o) && PyTuple_GET_SIZE(o) >= 3)
        return as_double(PyTuple_GET_ITEM(o, 0), out) && as_double(PyTuple_GET_ITEM(o, 1), out + 1) &&
               as_double(PyTuple_GET_ITEM(o, 2), out + 2);
    PyObject *seq = PySequence_Fast(o, "");
    if (!seq) {
        PyErr_Clear();
        return 0;
    }
    int ok = PySequence_Fast_GET_SIZE(seq) >= 3;
    for (int i = 0; ok && i < 3; i++) ok = as_double(PySequence_Fast_GET_ITEM(seq, i), out + i);
    Py_DECREF(seq);
    return ok;
}

static int attr_vec3(PyObject *o, int name, double *out) {
    PyObject *a = get(o, name);
    if (!a) {
        PyErr_Clear();
        return 0;
    }
    int ok = vec3(a, out);
    Py_DECREF(a);
    return ok;
}

static int attr_double(PyObject *o, int name, double *out) {
    PyObject *a = get(o, name);
    if (!a) {
        PyErr_Clear();
        return 0;
    }
    int ok = as_double(a, out);
    Py_DECREF(a);
    return ok;
}

static int pack(PyObject *scene, Packed *p) {
    p->have_view = 0;
    PyObject *bodies = get(scene, A_BODIES);
    if (!bodies) {
        PyErr_Clear();
        return 0;
    }
    PyObject *seq = PySequence_Fast(bodies, "");
    Py_DECREF(bodies);
    if (!seq) {
        PyErr_Clear();
        return 0;
    }
    Py_ssize_t n = PySequence_Fast_GET_SIZE(seq);
    int ok = n <= MAX_BODIES;
    p->n = (int)n;
    for (Py_ssize_t i = 0; ok && i < n; i++) {
        PyObject *b = PySequence_Fast_GET_ITEM(seq, i);
        PyObject *k = get(b, A_KIND);
        if (!k) {
            PyErr_Clear();
            ok = 0;
            break;
        }
        long kv = PyLong_AsLong(k);
        Py_DECREF(k);
        if (kv == -1 && PyErr_Occurred()) {
            PyErr_Clear();
            ok = 0;
            break;
        }
        p->kinds[i] = (int32_t)kv;
        ok = attr_vec3(b, A_POSITION, p->pos + 3 * i) && attr_double(b, A_SIZE, p->size + i) &&
             attr_vec3(b, A_COLOR, p->color + 3 * i) && attr_double(b, A_REFLECTIVITY, p->refl + i);
    }
    Py_DECREF(seq);
    if (!ok) return 0;
    PyObject *light = get(scene, A_LIGHT);
    if (!light) {
        PyErr_Clear();
        return 0;
    }
    ok = attr_vec3(light, A_POSITION, p->light_pos) && attr_vec3(light, A_COLOR, p->light_color) &&
         attr_double(light, A_RADIUS, &p->light_radius);
    Py_DECREF(light);
    if (!ok || !attr_double(scene, A_AMBIENT, &p->ambient) || !attr_double(scene, A_MAX_REFL, &p->max_refl))
        return 0;
    PyObject *sky = get(scene, A_SKYBOX);
    if (!sky) PyErr_Clear();
    if (!sky || sky == Py_None) {
        Py_XDECREF(sky);
        p->sky = g_no_sky;
        p->sky_w = p->sky_h = 1;
        p->has_sky = 0;
        return 1;
    }
    double w = 0, h = 0;
    PyObject *tex = get(sky, A_TEXELS);
    ok = tex && attr_double(sky, A_WIDTH, &w) && attr_double(sky, A_HEIGHT, &h);
    Py_DECREF(sky);
    if (!tex) PyErr_Clear();
    if (ok && PyObject_GetBuffer(tex, &p->sky_view, PyBUF_C_CONTIGUOUS | PyBUF_FORMAT) == 0) {
        p->have_view = 1;
        const char *f = p->sky_view.format;
        ok = f && (f[0] == 'f' || ((f[0] == '<' || f[0] == '=') && f[1] == 'f')) && f[f[0] == 'f' ? 1 : 2] == 0 &&
             p->sky_view.itemsize == 4 && p->sky_view.len == (Py_ssize_t)(12 * (Py_ssize_t)w * (Py_ssize_t)h);
    } else {
        PyErr_Clear();
        ok = 0;
    }
    Py_XDECREF(tex);
    if (!ok) return 0;
    p->sky = (const float *)p->sky_view.buf;
    p->sky_w = (int32_t)w;
    p->sky_h = (int32_t)h;
    p->has_sky = 1;
    return 1;
}

static void unpack(Packed *p) {
    if (p->have_view) PyBuffer_Release(&p->sky_view);
    p->have_view = 0;
}

static PyObject *set_entry_points(PyObject *self, PyObject *args) {
    unsigned long long r = 0, a = 0;
    if (!PyArg_ParseTuple(args, "KK", &r, &a)) return NULL;
    g_render = (render_fn)(uintptr_t)r;
    g_async = (async_fn)(uintptr_t)a;
    Py_RETURN_NONE;
}

/* render(ctx, pixels, radiance, width, height, cam_position, yaw, pitch, vdist, scene,
 *        samples, bounces, n_parts, precision) -> rc, or None (take the generic path) */
static PyObject *render(PyObject *self, PyObject *args) {
    unsigned long long ctx, pixels, radiance;
    int w, h, samples, bounces, n_parts, prec;
    PyObject *campos, *scene;
    double yaw, pitch, vdist, cam[3];
    if (!PyArg_ParseTuple(args, "KKKiiOdddOiiii", &ctx, &pixels, &radiance, &w, &h, &campos, &yaw, &pitch, &vdist,
                          &scene, &samples, &bounces, &n_parts, &prec))
        return NULL;
    if (!g_render || !vec3(campos, cam)) Py_RETURN_NONE;
    Packed *p = &g_packed;  /* per thread: the GIL is released while the arrays are in use */
    if (!pack(scene, p)) {
        unpack(p);
        Py_RETURN_NONE;
    }
    int rc;
    Py_BEGIN_ALLOW_THREADS rc = g_render((void *)(uintptr_t)ctx, (uint32_t *)(uintptr_t)pixels,
                                         (void *)(uintptr_t)radiance, w, h, cam, yaw, pitch, vdist, p->n, p->kinds,
                                         p->pos, p->size, p->color, p->refl, p->light_pos, p->light_radius,
                                         p->light_color, p->ambient, p->max_refl, p->sky, p->sky_w, p->sky_h,
                                         p->has_sky, samples, bounces, n_parts, prec);
    Py_END_ALLOW_THREADS unpack(p);
    return PyLong_FromLong(rc);
}

/* render_async(ctx, slot, pixels, width, height, cam_position, yaw, pitch, vdist, scene,
 *              samples, bounces, precision) -> rc, or None */
static PyObject *render_async(PyObject *self, PyObject *args) {
    unsigned long long ctx, pixels;
    int slot, w, h, samples, bounces, prec;
    PyObject *campos, *scene;
    double yaw, pitch, vdist, cam[3];
    if (!PyArg_ParseTuple(args, "KiKiiOdddOiii", &ctx, &slot, &pixels, &w, &h, &campos, &yaw, &pitch, &vdist, &scene,
                          &samples, &bounces, &prec))
        return NULL;
    if (!g_async || !vec3(campos, cam)) Py_RETURN_NONE;
    Packed *p = &g_packed;
    if (!pack(scene, p)) {
        unpack(p);
        Py_RETURN_NONE;
    }
    int rc;
    Py_BEGIN_ALLOW_THREADS rc = g_async((void *)(uintptr_t)ctx, slot, (uint32_t *)(uintptr_t)pixels, w, h, cam, yaw,
                                        pitch, vdist, p->n, p->kinds, p->pos, p->size, p->color, p->refl,
                                        p->light_pos, p->light_radius, p->light_color, p->ambient, p->max_refl,
                                        p->sky, p->sky_w, p->sky_h, p->has_sky, samples, bounces, prec);
    Py_END_ALLOW_THREADS unpack(p);
    return PyLong_FromLong(rc);
}

static PyMethodDef methods[] = {
    {"set_entry_points", set_entry_points, METH_VARARGS, "addresses of rt_render_v1 and rt_render_async_v1"},
    {"render", render, METH_VARARGS, "rt_render_v1 on a duck-typed reference Scene"},
    {"render_async", render_async, METH_VARARGS, "rt_render_async_v1 on a duck-typed reference Scene"},
    {NULL, NULL, 0, NULL}};

static struct PyModuleDef module = {PyModuleDef_HEAD_INIT, "_pyfast", NULL, -1, methods};

PyMODINIT_FUNC PyInit__pyfast(void) {
    for (int i = 0; i < A_N; i++)
        if (!g_attr[i] && !(g_attr[i] = PyUnicode_InternFromString(g_attr_names[i]))) return NULL;
    return PyModule_Create(&module);
}
